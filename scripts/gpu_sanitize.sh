# compute-sanitizer (memcheck, synccheck, racecheck) over small tests of every kernel:
# the filter path (guess, filter, refine), the fixup kernel, the fused row kernel (incl.
# the snap branch and the second pass), the cluster kernel at G = 2/4/8 (DSMEM), the radix
# baselines.  -> gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
SEL="filter_path_small_k and 100 or events_entry_point_filter_path or fixup_kernel_short_lists or snap_branch or cluster_rows and 20001 or guess_overshoot and 20000 or radix2_baseline_exact and 20001"
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_phase2.py -q \
    -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.log | tail -4
done
