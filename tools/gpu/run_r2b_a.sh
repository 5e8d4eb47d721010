cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_a.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_errors.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_a.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-helmholtz --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_a.log
timeout 600 python tools/helm_config3.py 6 > gpurun_out/helm_a.log 2>&1
echo "helm rc=$?" >> gpurun_out/helm_a.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_h_ctr|k_h_p2w" -c 2 -o gpurun_out/hctr_a python tools/helm_config3.py 6 > gpurun_out/ncu_hctr_a.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_hctr_a.log
