"""Sweep the collect-threshold width sigma (T_c = pmean - sigma * sd) on a bench config:
time per step, and the per-row stats (raises, f(T_c), fallbacks).
usage: python scripts/sigma_sweep.py [--config cfg2] [--sigmas 0.5,0.4,...]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--sigmas", default="0.5,0.45,0.4,0.35,0.3,0.25")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--stride", type=int, default=0, help="guess_stride option (0 = library default)")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
batches = [bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.splitmix64(synth.BASE_SEED, b),
                                   draft=cfg["draft"]) for b in range(3)]
torch.cuda.synchronize()
R = batches[0]["R"]
out = torch.empty((R, bench.K), dtype=torch.int32, device=dev)
F = gvr.STATS_FIELDS
for s in [float(x) for x in args.sigmas.split(",")]:
    opt = gvr.GvrOptions(s, 0, 0, args.stride)
    stats = []
    for b in batches:
        _, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out, values=False,
                               options=opt)
        stats.append(st.cpu().numpy())
    st = np.concatenate(stats)
    def step(i):
        b = batches[i % 3]
        gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out, values=False, stats=False,
                    options=opt)
    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.steps
    col = lambda n: st[:, F.index(n)]
    bc = col("buffer_count")
    print(f"stride {args.stride} sigma {s:4.2f}: {us:7.1f} us/step  raises/row {col('raises').mean():.2f} (rows>0 {np.mean(col('raises') > 0):.2f})"
          f"  f(Tc) p10/50/90 {np.percentile(bc, 10):.0f}/{np.percentile(bc, 50):.0f}/{np.percentile(bc, 90):.0f}"
          f"  fallback {np.mean(col('done_kind') >= 2):.3f}  secant {col('secant_iters').mean():.2f}"
          f"  snap {col('snap_iters').mean():.2f}  cand {col('cand_count').mean():.0f}", flush=True)
