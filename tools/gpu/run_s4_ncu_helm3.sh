cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
k=k_h_m2l_pas
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 -f -o gpurun_out/helm3_$k python tools/helm_config3.py 6 > gpurun_out/ncu_helm3_$k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_helm3_$k.log
ncu -i gpurun_out/helm3_$k.ncu-rep --page raw --csv > gpurun_out/helm3_${k}_raw.csv 2>/dev/null
