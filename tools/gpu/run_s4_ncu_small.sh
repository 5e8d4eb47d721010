cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_s4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_l2qbxl3|k_p2l3|k_p2m" -c 3 -f -o gpurun_out/small_s4 python tools/apply_once.py 1 1 > gpurun_out/ncu_small_s4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_small_s4.log
ncu -i gpurun_out/small_s4.ncu-rep --page raw --csv > gpurun_out/small_s4_raw.csv 2>/dev/null
