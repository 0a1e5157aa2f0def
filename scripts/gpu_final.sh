# Round measurement set: full parity suite, smoke, bench lines (default cfg2 with e2e and
# cpu_baseline; cfg1/cfg3/cfg4/cfg5; row path cfg2; reference arm), batch-1 latency sweep,
# ncu summaries of the filter-path kernels and the ncu launch list.  -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log | head -c 3000; echo
for c in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_$c.log 2>&1; tail -n 1 gpurun_out/bench_$c.log | head -c 400; echo; done
timeout 900 python bench.py --path row --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_row.log 2>&1; tail -n 1 gpurun_out/bench_row.log | head -c 300; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; tail -n 1 gpurun_out/bench_reference.log | head -c 300; echo
timeout 900 python scripts/latency_sweep.py > gpurun_out/latency_sweep.jsonl 2>&1; cut -c 1-200 gpurun_out/latency_sweep.jsonl
for kn in gvr_filter_kernel gvr_refine_kernel gvr_guess_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o gpurun_out/prof_$kn -f python scripts/prof_kernels.py > gpurun_out/ncu_$kn.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_$kn.ncu-rep > gpurun_out/summary_$kn.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'gvr_|radix_' --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/traffic_from_ncu.py gvr_cfg2=gpurun_out/prof_gvr_filter_kernel.ncu-rep refine_cfg2=gpurun_out/prof_gvr_refine_kernel.ncu-rep guess_cfg2=gpurun_out/prof_gvr_guess_kernel.ncu-rep > gpurun_out/traffic.log 2>&1; cat gpurun_out/traffic.log
cp profiles/traffic.json gpurun_out/traffic.json
