cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_u.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_u.log
grep -q "smoke rc=0" gpurun_out/smoke_u.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_u.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_u.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline --no-config4 > gpurun_out/bench_u.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_u.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_u.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near_qbx" -c 1 -o gpurun_out/near_u python tools/apply_once.py 1 1 > gpurun_out/ncu_u.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_u.log
