# Round measurement set: smoke, full parity suite, bench lines (default cfg2 with e2e and
# cpu_baseline; cfg1/cfg3/cfg4/cfg5; row path cfg2; radix2; reference arm), batch-1 latency
# sweep, worst cases, ncu --set full of the filter-path kernels (summaries + raw metrics:
# passes, bank conflicts), the ncu launch list, traffic.json.  -> gpurun_out/final/
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --steps 50 --warmup 5 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -n 1 $O/bench_cfg2.json | head -c 600; echo
for c in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; tail -n 1 $O/bench_$c.json | head -c 300; echo; done
timeout 900 python bench.py --path row --steps 50 --warmup 5 --no-e2e --no-cpu > $O/bench_rowpath.json 2>&1
timeout 900 python bench.py --impl radix2 --steps 50 --warmup 5 --no-e2e --no-cpu > $O/bench_radix2.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; tail -n 1 $O/bench_reference.json | head -c 300; echo
timeout 900 python scripts/latency_sweep.py > $O/latency_sweep.jsonl 2>&1
timeout 900 python scripts/worst_cases.py > $O/worst_cases.jsonl 2>&1
for kn in gvr_filter_kernel gvr_refine_kernel gvr_guess_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o $O/prof_$kn -f python scripts/prof_kernels.py > $O/ncu_$kn.log 2>&1
  python scripts/ncu_summary.py $O/prof_$kn.ncu-rep > $O/summary_$kn.txt 2>&1
  python scripts/ncu_raw_metrics.py $O/prof_$kn.ncu-rep 195200000 >> $O/summary_$kn.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'gvr_|radix' --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
python scripts/traffic_from_ncu.py gvr_cfg2=$O/prof_gvr_filter_kernel.ncu-rep refine_cfg2=$O/prof_gvr_refine_kernel.ncu-rep guess_cfg2=$O/prof_gvr_guess_kernel.ncu-rep > $O/traffic.log 2>&1; cat $O/traffic.log
cp profiles/traffic.json $O/traffic.json
for kn in gvr_filter_kernel gvr_refine_kernel gvr_guess_kernel; do echo "== $kn"; tail -22 $O/summary_$kn.txt; done
timeout 300 python scripts/filter_timeline.py cfg2 > $O/cta_timeline_cfg2.log 2>&1
timeout 300 python scripts/filter_timeline.py cfg4 > $O/cta_timeline_cfg4.log 2>&1
timeout 300 python scripts/refine_timing.py > $O/refine_timing_cfg2.log 2>&1
