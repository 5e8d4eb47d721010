cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_shard.py tests/test_direct_qbx.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider -k "not helmholtz_m2l_variant" > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_b.log
timeout 300 python tools/apply_once.py 1 2 > gpurun_out/plain_b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv python tools/apply_once.py 1 2 > gpurun_out/ncu_b.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_b.log
