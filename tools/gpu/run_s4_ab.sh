# A/B over the libraries in variants/: per-stage times of config 1, interleaved
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/ab_s4.log
for rep in 1 2; do
for v in $VARIANTS; do
cp variants/lib_$v.so paper_1805_06106_b200/libqbxg.so
echo "$v $(timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/ab_s4.log
done
done
