cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp gpurun_out/lib_w8.so paper_1805_06106_b200/libqbxg.so
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1
echo "rc=$?" >> gpurun_out/smoke_s3.log
