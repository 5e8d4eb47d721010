cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
true
echo "pytest rc=$?" >> gpurun_out/pytest_o.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline --no-config4 > gpurun_out/bench_o.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_o.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_o.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_o.csv python tools/apply_once.py 1 1 > gpurun_out/ncu_o.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_o.log
