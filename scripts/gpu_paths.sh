# Both batch paths on every multi-wave config (bench lines), after a quick parity check.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "filter or full_size or split or events" > gpurun_out/pytest_quick.log 2>&1; echo "quick rc=$?" >> gpurun_out/pytest_quick.log
tail -n 2 gpurun_out/pytest_quick.log
for c in cfg2 cfg4 cfg5; do for p in filter row; do
timeout 600 python bench.py --config $c --path $p --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_${c}_$p.log 2>&1
tail -n 1 gpurun_out/bench_${c}_$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $p', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_us_per_launch'], d['speedup_vs_radix'])"
done; done
