#!/bin/bash
# ncu --set full of one kernel (regex $1) on config $2 (default cfg2) + its SASS source page.
kn=${1:-gvr_refine_kernel}; cfg=${2:-cfg2}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o gpurun_out/prof_$kn -f python scripts/prof_kernels.py --config $cfg > gpurun_out/ncu_$kn.log 2>&1
ncu -i gpurun_out/prof_$kn.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$kn.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof_$kn.ncu-rep > gpurun_out/summary_$kn.txt 2>&1
cat gpurun_out/summary_$kn.txt
