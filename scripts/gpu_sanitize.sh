# compute-sanitizer (memcheck, synccheck, racecheck) over small filter-path and row-path
# parity tests.  -> gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "filter_path_small_k and 100 or events_entry_point_filter_path" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.log | tail -4
done
