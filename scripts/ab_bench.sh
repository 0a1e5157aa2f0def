#!/bin/bash
# A/B of library builds on one box: each .so copied over the in-tree lib in turn, bench.py
# (no e2e / cpu legs) on the given configs, ROUNDS interleaved rounds; prints ms_per_step.
# Usage: ROUNDS=3 CFGS="cfg2 cfg4" bash scripts/ab_bench.sh a.so b.so ...
cd ${GRAFT_REPO_ROOT:-.}
cp paper_2604_22312_b200/libgvrtopk.so /tmp/lib_keep.so
for r in $(seq ${ROUNDS:-3}); do
  for l in "$@"; do
    cp $l paper_2604_22312_b200/libgvrtopk.so
    for c in ${CFGS:-cfg2}; do
      ms=$(python bench.py --config $c --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_us_per_launch'])")
      echo "round $r $l $c $ms"
    done
  done
done
cp /tmp/lib_keep.so paper_2604_22312_b200/libgvrtopk.so
