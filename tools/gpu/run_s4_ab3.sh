cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/ab_s4.log gpurun_out/pytest_ab.log
for rep in 1 2; do
for v in $VARIANTS; do
cp variants/lib_$v.so paper_1805_06106_b200/libqbxg.so
echo "$v $(timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/ab_s4.log
done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_direct_qbx.py tests/test_gpu_errors.py tests/test_golden.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
