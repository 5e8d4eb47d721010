cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/helm_config3.py 5 > gpurun_out/helm_w.log 2>&1
echo "rc=$?" >> gpurun_out/helm_w.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_h_ctr" -c 2 -o gpurun_out/helm_w python tools/helm_config3.py 5 > gpurun_out/ncu_w.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_w.log
