# ncu --set full of the batch filter path's kernels on cfg2 (one launch each) + launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
for kn in gvr_filter_kernel gvr_refine_kernel gvr_guess_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o gpurun_out/prof_$kn -f python scripts/prof_kernels.py > gpurun_out/ncu_$kn.log 2>&1
  ncu -i gpurun_out/prof_$kn.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$kn.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/prof_$kn.ncu-rep > gpurun_out/summary_$kn.txt 2>&1
  python scripts/ncu_stalls.py gpurun_out/sass_$kn.csv paper_2604_22312_b200/libgvrtopk.so $kn > gpurun_out/stalls_$kn.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'gvr_|radix_' --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
for kn in gvr_filter_kernel gvr_refine_kernel gvr_guess_kernel; do echo "== $kn"; cat gpurun_out/summary_$kn.txt; head -25 gpurun_out/stalls_$kn.txt; done
