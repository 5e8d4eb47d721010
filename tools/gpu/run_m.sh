cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_m.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_m.log
