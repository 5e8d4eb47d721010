cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_helmholtz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_y.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_y.log
timeout 600 python tools/helm_config3.py 6 > gpurun_out/helm_y.log 2>&1
echo "rc=$?" >> gpurun_out/helm_y.log
