cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_i.log 2> gpurun_out/bench_i.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))" >> gpurun_out/bench_i.log
