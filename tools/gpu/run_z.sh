cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_z.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2l3|k_l2qbxl3|k_p2m" -c 3 -o gpurun_out/small_z python tools/apply_once.py 1 1 > gpurun_out/ncu_z.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_z.log
