cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r.log
timeout 900 python bench.py > gpurun_out/bench_r.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_r.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_r.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r.csv python tools/apply_once.py 1 1 > gpurun_out/ncu_r.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r.log
