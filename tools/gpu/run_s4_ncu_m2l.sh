cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/apply_once.py 1 1 > gpurun_out/plain_s4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tg -c 1 -f -o gpurun_out/m2l_s4 python tools/apply_once.py 1 1 > gpurun_out/ncu_s4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_s4.log
ncu -i gpurun_out/m2l_s4.ncu-rep --page source --csv > gpurun_out/m2l_s4_source.csv 2>/dev/null
