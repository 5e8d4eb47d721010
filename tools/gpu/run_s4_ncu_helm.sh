cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in k_h_m2l_pas k_h_ctr; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/helm_$k python tools/helm_config3.py 6 > gpurun_out/ncu_helm_$k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_helm_$k.log
ncu -i gpurun_out/helm_$k.ncu-rep --page raw --csv > gpurun_out/helm_${k}_raw.csv 2>/dev/null
done
