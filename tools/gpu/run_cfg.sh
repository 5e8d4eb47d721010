cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/config_run.py 0 1 2 3 > gpurun_out/configs_r02.jsonl 2> gpurun_out/configs_r02.err
echo "rc=$?" >> gpurun_out/configs_r02.err
timeout 1500 python tools/config4_run.py > gpurun_out/config4_r02.jsonl 2> gpurun_out/config4_r02.err
echo "rc=$?" >> gpurun_out/config4_r02.err
