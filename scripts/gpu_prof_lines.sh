#!/bin/bash
# ncu --set full of the refine and guess kernels (cfg2) + instructions per source line
# (ncu_instr_lines.py) and the kernel trace.  -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python scripts/kernel_trace.py > gpurun_out/trace.log 2>&1
for kn in ${KERNELS:-gvr_refine_kernel gvr_guess_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o gpurun_out/prof_$kn -f python scripts/prof_kernels.py > gpurun_out/ncu_$kn.log 2>&1
  ncu -i gpurun_out/prof_$kn.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$kn.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/prof_$kn.ncu-rep > gpurun_out/summary_$kn.txt 2>&1
  python scripts/ncu_instr_lines.py gpurun_out/sass_$kn.csv paper_2604_22312_b200/libgvrtopk.so $kn 488 45 > gpurun_out/lines_$kn.txt 2>&1
done
