cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_c.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_m2l_fused -c 1 -o gpurun_out/m2l_fused_c python tools/apply_once.py 1 1 > gpurun_out/ncu_c.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c.log
