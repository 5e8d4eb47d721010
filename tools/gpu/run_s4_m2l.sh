cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_m2l.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m2l.log
for rep in 1 2; do
echo "$(timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/st_m2l.log
done
