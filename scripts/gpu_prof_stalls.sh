#!/bin/bash
# ncu --set full of the given kernels (default: guess, refine) on config $CFG (default cfg2),
# one launch each, then per-source-line stall attribution.  Usage: bash scripts/gpu_prof_stalls.sh [kernel...]
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
cfg=${CFG:-cfg2}
for kn in ${@:-gvr_guess_kernel gvr_refine_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o gpurun_out/prof_$kn -f python scripts/prof_kernels.py --config $cfg > gpurun_out/ncu_$kn.log 2>&1
  ncu -i gpurun_out/prof_$kn.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$kn.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/prof_$kn.ncu-rep > gpurun_out/summary_$kn.txt 2>&1
  python scripts/ncu_stalls.py gpurun_out/sass_$kn.csv paper_2604_22312_b200/libgvrtopk.so $kn 40 > gpurun_out/stalls_$kn.txt 2>&1
done
