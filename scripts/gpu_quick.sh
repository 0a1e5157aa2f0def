cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "filter or full_size or split or events" > gpurun_out/pytest_quick.log 2>&1; echo "quick rc=$?" >> gpurun_out/pytest_quick.log
tail -n 4 gpurun_out/pytest_quick.log
timeout 300 python scripts/refine_timing.py > gpurun_out/refine_timing.log 2>&1; cat gpurun_out/refine_timing.log | tail -20
