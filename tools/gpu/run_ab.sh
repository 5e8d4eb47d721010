cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
for v in 2cta dual; do
cp gpurun_out/lib_$v.so paper_1805_06106_b200/libqbxg.so
echo "$v $(timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/ab.log
done
done
