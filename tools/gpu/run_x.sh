cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/stage_times.py 1 5 > gpurun_out/st_x0.log 2>&1
QBXG_OVERLAP=1 timeout 300 python tools/stage_times.py 1 5 > gpurun_out/st_x1.log 2>&1
