# A/B of the guess gather fetch size (L2::64B hint vs none): guess kernel time per config.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 64 32; do
  if [ $v = 32 ]; then sed -i 's/ld.global.nc.L1::no_allocate.L2::64B.f32/ld.global.nc.L1::no_allocate.f32/' paper_2604_22312_b200/csrc/gvr_kernel.cuh; fi
  GVR_FORCE_BUILD=1 python __graft_entry__.py > gpurun_out/build_$v.log 2>&1
  for c in cfg2 cfg4; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_fetch${v}_$c.log 2>&1
    tail -n 1 gpurun_out/bench_fetch${v}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fetch$v $c', d['value'], d['ms_per_step'], d['kernel_us_per_launch'], d['passes_per_row'])"
  done
done
