#!/bin/bash
# ncu --set full of one kernel (KN) for each library in LIBS (ab/<lib>): summary + per-line instructions.
cd ${GRAFT_REPO_ROOT:-.}
LIB=paper_2604_22312_b200/libgvrtopk.so
cp $LIB /tmp/lib_keep.so
for l in ${LIBS}; do
  cp ab/$l.so $LIB
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KN} -s 2 -c 1 -o gpurun_out/prof_${KN}_$l -f python scripts/prof_kernels.py > /dev/null 2>&1
  ncu -i gpurun_out/prof_${KN}_$l.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${KN}_$l.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/prof_${KN}_$l.ncu-rep > gpurun_out/summary_${KN}_$l.txt 2>&1
  python scripts/ncu_instr_lines.py gpurun_out/sass_${KN}_$l.csv $LIB ${KN} 488 30 > gpurun_out/lines_${KN}_$l.txt 2>&1
  echo "== $l"; head -16 gpurun_out/summary_${KN}_$l.txt; head -12 gpurun_out/lines_${KN}_$l.txt
done
cp /tmp/lib_keep.so $LIB
