cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/helm_ab.log
timeout 1500 python -m pytest tests/test_helmholtz.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "helm or Helm" > gpurun_out/pytest_helm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_helm.log
for v in $VARIANTS; do
cp variants/lib_$v.so paper_1805_06106_b200/libqbxg.so
echo "== $v" >> gpurun_out/helm_ab.log
timeout 600 python tools/helm_config3.py 6 >> gpurun_out/helm_ab.log 2>&1
done
