cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_shard.py tests/test_gpu_errors.py tests/test_direct_qbx.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "not helmholtz_m2l_variant and not helmholtz_config3" > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_e.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline > gpurun_out/bench_e.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_e.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_e.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_near_qbx -c 1 -o gpurun_out/near_e python tools/apply_once.py 1 1 > gpurun_out/ncu_e.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_e.log
