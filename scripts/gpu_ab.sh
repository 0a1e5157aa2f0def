#!/bin/bash
# A/B of refine-kernel variants (ab/*.so): quick filter-path parity per variant, refine
# phase timing, then interleaved bench rounds.  Usage: VARIANTS="A B" bash scripts/gpu_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIB=paper_2604_22312_b200/libgvrtopk.so
for v in ${VARIANTS:-A}; do
  cp ab/$v.so $LIB
  timeout 600 python -m pytest tests -m gpu -q -x -k "${TESTK:-filter or full_size or split or events or tie or trivial or short}" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -n 2 gpurun_out/pytest_$v.log
  timeout 300 python scripts/refine_timing.py > gpurun_out/rt_$v.log 2>&1; grep -E "span|cycles|serialised|whole call" gpurun_out/rt_$v.log
done
ROUNDS=${ROUNDS:-2} CFGS="${CFGS:-cfg2 cfg4}" bash scripts/ab_bench.sh $(for v in ${BASE:-base} ${VARIANTS:-A}; do echo ab/$v.so; done)
# optional: ncu source-level profile of the refine kernel for variant $PROF
if [ -n "$PROF" ]; then
  cp ab/$PROF.so $LIB
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gvr_refine_kernel -s 2 -c 1 -o gpurun_out/prof_refine_$PROF -f python scripts/prof_kernels.py > gpurun_out/ncu_refine_$PROF.log 2>&1
  ncu -i gpurun_out/prof_refine_$PROF.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_refine_$PROF.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/prof_refine_$PROF.ncu-rep > gpurun_out/summary_refine_$PROF.txt 2>&1
  python scripts/ncu_instr_lines.py gpurun_out/sass_refine_$PROF.csv $LIB gvr_refine_kernel 488 45 > gpurun_out/lines_refine_$PROF.txt 2>&1
  head -30 gpurun_out/summary_refine_$PROF.txt
fi
