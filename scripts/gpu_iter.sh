# GPU iteration: build, targeted parity tests, refine timing, bench lines (both batch
# paths), then the full -m gpu suite.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "filter or full_size or split or events" > gpurun_out/pytest_quick.log 2>&1; echo "quick rc=$?" >> gpurun_out/pytest_quick.log
tail -n 3 gpurun_out/pytest_quick.log
timeout 300 python scripts/refine_timing.py > gpurun_out/refine_timing.log 2>&1; tail -n 16 gpurun_out/refine_timing.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_filter.log 2>&1; tail -n 1 gpurun_out/bench_filter.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('filter', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_us_per_launch'], d['passes_per_row'])"
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --path row > gpurun_out/bench_row.log 2>&1; tail -n 1 gpurun_out/bench_row.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('row', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_us_per_launch'])"
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
