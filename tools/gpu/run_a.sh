cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/nproc_a.txt; lscpu | head -20 >> gpurun_out/nproc_a.txt
timeout 1500 python -m pytest tests -m gpu -q -k "not helmholtz_config3_settings_level3" -p no:cacheprovider --durations=15 > gpurun_out/pytest_a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_a.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_a.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_a.log 2>&1
echo "ref rc=$?" >> gpurun_out/ref_a.log
