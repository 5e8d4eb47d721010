cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_direct_qbx.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_b.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "config1" > gpurun_out/pytest_full_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full_b.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near_qbx" -c 1 -o gpurun_out/near_b python tools/apply_once.py 1 1 > gpurun_out/ncu_near_b.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_near_b.log
