#!/bin/bash
# Interleaved A/B over (library, environment) pairs: ARMS="H.so: P.so:GVR_POOL_PCT=0" (ab/<lib>,
# env after the colon), ROUNDS rounds of bench.py on CFGS; prints ms_per_step + kernels.
cd ${GRAFT_REPO_ROOT:-.}
LIB=paper_2604_22312_b200/libgvrtopk.so
cp $LIB /tmp/lib_keep.so
for r in $(seq ${ROUNDS:-2}); do
  for a in ${ARMS}; do
    l=${a%%:*}; e=${a#*:}
    cp ab/$l $LIB
    for c in ${CFGS:-cfg2}; do
      ms=$(env X=1 $e python bench.py --config $c --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_us_per_launch'], {k: round(v, 2) for k, v in (d.get('passes_per_row') or {}).items() if k in ('secant_mean', 'cand_mean')})")
      echo "round $r $a $c $ms"
    done
  done
done
cp /tmp/lib_keep.so $LIB
