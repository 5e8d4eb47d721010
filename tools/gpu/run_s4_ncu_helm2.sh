cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
k=k_h_ctr
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 -f -o gpurun_out/helm2_$k python tools/helm_config3.py 6 > gpurun_out/ncu_helm2_$k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_helm2_$k.log
ncu -i gpurun_out/helm2_$k.ncu-rep --page raw --csv > gpurun_out/helm2_${k}_raw.csv 2>/dev/null
