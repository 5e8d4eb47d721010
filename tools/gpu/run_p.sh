cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_p.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_p.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_p.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_p.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_p.log
timeout 1200 python bench.py > gpurun_out/bench_p.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_p.log
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_p.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref_p.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_p.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_p.csv python tools/apply_once.py 1 1 > gpurun_out/ncu_p.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_p.log
