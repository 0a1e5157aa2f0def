# One GPU session: parity, profiles (gvr, guess, radix, launch list), bench lines for
# every config, batch-1 latency sweep.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
bash scripts/gpu_prof.sh > /dev/null 2>&1
for c in cfg1 cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_$c.log 2>&1; tail -n 1 gpurun_out/bench_$c.log | head -c 400; echo; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; tail -n 1 gpurun_out/bench_reference.log | head -c 400; echo
timeout 900 python scripts/latency_sweep.py > gpurun_out/latency_sweep.jsonl 2>&1; cat gpurun_out/latency_sweep.jsonl | cut -c 1-300
tail -n 1 gpurun_out/bench.log | head -c 600
