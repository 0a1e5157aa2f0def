#!/bin/bash
# On the GPU box: the GPU test suite (-x) then bench.py lines for the given configs
# (default cfg2 cfg4 cfg5), results under gpurun_out/.  Usage: bash scripts/gpu_check.sh [notest] [cfg...]
mkdir -p gpurun_out
if [ "$1" != "notest" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
else
  shift
fi
cfgs="${@:-cfg2 cfg4 cfg5}"
for c in $cfgs; do
  python bench.py --config $c --no-e2e --no-cpu > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err || tail -5 gpurun_out/b_$c.err
done
