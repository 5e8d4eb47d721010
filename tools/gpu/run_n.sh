cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider -k "not helmholtz" > gpurun_out/pytest_n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_n.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline --no-config4 > gpurun_out/bench_n.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_n.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_n.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n.csv python tools/apply_once.py 1 1 > gpurun_out/ncu_n.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_n.log
