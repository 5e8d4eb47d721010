cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_h.log
/usr/bin/time -v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_h.log 2> gpurun_out/bench_h.err
echo "bench rc=$?" >> gpurun_out/bench_h.log
