cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_s4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_s4.log
timeout 1200 python bench.py > gpurun_out/bench_s4.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_s4.log
timeout 600 python tools/helm_config3.py 6 > gpurun_out/helm3_s4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/helm_launches_s4.csv python tools/helm_config3.py 6 > gpurun_out/ncul_helm_s4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncul_helm_s4.log
