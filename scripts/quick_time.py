"""A/B timing of several builds of libgvrtopk.so in one process on the same inputs.
usage: python scripts/quick_time.py [--config cfg2] lib1.so lib2.so ..."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, synth

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
batches = [bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.splitmix64(synth.BASE_SEED, b),
                                   draft=cfg["draft"]) for b in range(3)]
torch.cuda.synchronize()
R = batches[0]["R"]
S = batches[0]["scores"].shape[1]
outs = [torch.empty((R, bench.K), dtype=torch.int32, device=dev) for _ in batches]
libs = []
for p in args.libs:
    l = ctypes.CDLL(os.path.abspath(p))
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    l.gvr_topk_batched.argtypes = [vp, i64, vp, i32, vp, i32, vp, vp]
    l.radix_topk_batched.argtypes = [vp, i64, vp, i32, i32, vp, vp]
    libs.append((p, l))
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)
ref = None
for rep in range(args.reps):
    for name, l in libs:
        for kind in ("gvr", "radix"):
            def step(i):
                b = batches[i % 3]
                if kind == "gvr":
                    rc = l.gvr_topk_batched(ctypes.c_void_p(b["scores"].data_ptr()), S, ctypes.c_void_p(b["row_lens"].data_ptr()), R,
                                            ctypes.c_void_p(b["prev"].data_ptr()), bench.K, ctypes.c_void_p(outs[i % 3].data_ptr()), sp)
                else:
                    rc = l.radix_topk_batched(ctypes.c_void_p(b["scores"].data_ptr()), S, ctypes.c_void_p(b["row_lens"].data_ptr()), R,
                                              bench.K, ctypes.c_void_p(outs[i % 3].data_ptr()), sp)
                assert rc == 0
            for i in range(5):
                step(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(args.steps):
                step(i)
            e1.record(st)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / args.steps * 1e3
            o = outs[0].cpu().numpy()
            if ref is None:
                ref = o
            ok = np.array_equal(o, ref)
            print(f"rep {rep} {os.path.basename(name):28s} {kind:5s} {us:8.1f} us/step  {R/us:.3f} Mrows/s  same_as_first={ok}", flush=True)
