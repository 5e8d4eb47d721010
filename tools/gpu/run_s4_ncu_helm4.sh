cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_h_p2w" --launch-skip 1 -c 1 -f -o gpurun_out/helm4_p2l python tools/helm_config3.py 6 > gpurun_out/ncu_helm4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_helm4.log
ncu -i gpurun_out/helm4_p2l.ncu-rep --page raw --csv > gpurun_out/helm4_p2l_raw.csv 2>/dev/null
