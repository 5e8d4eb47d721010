cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_t.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_t.log
grep -q "smoke rc=0" gpurun_out/smoke_t.log || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_errors.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_t.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline --no-config4 > gpurun_out/bench_t.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_t.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_t.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_tg|k_near_qbx" -c 2 -o gpurun_out/top_t python tools/apply_once.py 1 1 > gpurun_out/ncu_t.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_t.log
