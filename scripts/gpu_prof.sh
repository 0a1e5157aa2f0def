cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gvr_topk_kernel -s 2 -c 1 -o gpurun_out/prof_gvr -f python scripts/prof_kernels.py > gpurun_out/ncu_gvr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:radix_topk_kernel -s 1 -c 1 -o gpurun_out/prof_radix -f python scripts/prof_kernels.py > gpurun_out/ncu_radix.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gvr_|radix_' --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gvr_guess_kernel -s 2 -c 1 -o gpurun_out/prof_guess -f python scripts/prof_kernels.py > gpurun_out/ncu_guess.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1
tail -n 3 gpurun_out/ncu_gvr.log gpurun_out/ncu_radix.log; tail -n 2 gpurun_out/bench.log
