#!/bin/bash
# iteration: filter-path parity subset, smoke, refine timing, bench cfg2/cfg4/cfg5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "filter or full_size or split or phase2 or high_alpha or ties or mtp or events or graph" > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
python scripts/refine_timing.py cfg2 > gpurun_out/refine_timing.log 2>&1; head -9 gpurun_out/refine_timing.log
bash scripts/gpu_check.sh notest ${@:-cfg2 cfg4 cfg5}
