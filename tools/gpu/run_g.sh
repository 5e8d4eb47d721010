cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_helmholtz.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py -m gpu -q -p no:cacheprovider -k "helm or Helm" --durations=10 > gpurun_out/pytest_g.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_g.log
timeout 600 python tools/helm_config3.py > gpurun_out/helm3_g.log 2>&1
echo "helm rc=$?" >> gpurun_out/helm3_g.log
