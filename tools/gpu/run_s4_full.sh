cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_s4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_s4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_s4.log
timeout 1200 python bench.py > gpurun_out/bench_s4.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_s4.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_s4.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s4.csv python tools/apply_once.py 1 1 > gpurun_out/ncul_s4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncul_s4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_tg|k_near_qbx" -c 2 -f -o gpurun_out/top_s4 python tools/apply_once.py 1 1 > gpurun_out/ncu_top_s4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_top_s4.log
ncu -i gpurun_out/top_s4.ncu-rep --page raw --csv > gpurun_out/top_s4_raw.csv 2>/dev/null
