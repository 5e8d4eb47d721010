cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_f.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_f.log
timeout 1200 python bench.py > gpurun_out/bench_f.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_f.log
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_f.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref_f.log
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_f.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_f.csv python tools/apply_once.py 1 1 > gpurun_out/ncu_f.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_f.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_tg|k_near_qbx" -c 2 -o gpurun_out/top_f python tools/apply_once.py 1 1 > gpurun_out/ncu_top_f.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_top_f.log
timeout 600 python tools/helm_config3.py 6 > gpurun_out/helm_f.log 2>&1
