cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/ov_s4.log
for rep in 1 2; do
echo "seq $(timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/ov_s4.log
echo "ovl $(QBXG_OVERLAP=1 timeout 300 python tools/stage_times.py 1 5 | tail -n 1)" >> gpurun_out/ov_s4.log
done
