cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gvr_topk_kernel -s 2 -c 1 -o gpurun_out/prof_gvr -f python scripts/prof_kernels.py > gpurun_out/ncu_gvr.log 2>&1
tail -2 gpurun_out/ncu_gvr.log
