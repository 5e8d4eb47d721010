cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_s4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_s4.log
timeout 1200 python bench.py > gpurun_out/bench_s4.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_s4.log
