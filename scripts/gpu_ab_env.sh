#!/bin/bash
# A/B of one library under environment settings: ENVS="GVR_POOL_PCT=0 GVR_POOL_PCT=20" —
# interleaved rounds of bench.py (no e2e / cpu legs) on CFGS; prints ms_per_step + kernels.
cd ${GRAFT_REPO_ROOT:-.}
for r in $(seq ${ROUNDS:-2}); do
  for e in ${ENVS:-X=1}; do
    for c in ${CFGS:-cfg2}; do
      ms=$(env $e python bench.py --config $c --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_us_per_launch'])")
      echo "round $r $e $c $ms"
    done
  done
done
