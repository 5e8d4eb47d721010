cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_h_near" -c 1 -f -o gpurun_out/helm5_near python tools/helm_config3.py 6 > gpurun_out/ncu_helm5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_helm5.log
ncu -i gpurun_out/helm5_near.ncu-rep --page raw --csv > gpurun_out/helm5_near_raw.csv 2>/dev/null
