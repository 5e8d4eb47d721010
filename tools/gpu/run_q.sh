cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_q.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_q.log
grep -q "smoke rc=0" gpurun_out/smoke_q.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline --no-config4 > gpurun_out/bench_q.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_q.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tg -c 1 -o gpurun_out/m2l_q python tools/apply_once.py 1 1 > gpurun_out/ncu_q.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_q.log
