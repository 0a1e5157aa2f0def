"""Global timeline of one GVR launch on a bench config: CTA start/end (globaltimer) per
row and SM, resident CTAs per SM over time, and the kernel times from CUDA events."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=0, help="bench batch index (seed splitmix64(BASE_SEED, i))")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
b = bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.splitmix64(synth.BASE_SEED, args.batch),
                           draft=cfg["draft"])
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for _ in range(3):
    flush.zero_()
    out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flush.zero_()
e0.record()
out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
e1.record()
torch.cuda.synchronize()
t = ts.cpu().numpy().astype(np.int64)
gs, ge, sm = t[:, 6], t[:, 7], t[:, 8]
t0 = gs.min()
gs, ge = (gs - t0) / 1e3, (ge - t0) / 1e3  # us
R = len(gs)
print(f"events: {e0.elapsed_time(e1)*1e3:.1f} us for the launch pair; CTA span {ge.max():.1f} us "
      f"(first start 0, last start {gs.max():.1f}, last end {ge.max():.1f})")
dur = ge - gs
print(f"row duration us: p10 {np.percentile(dur,10):.1f} p50 {np.median(dur):.1f} p90 {np.percentile(dur,90):.1f} max {dur.max():.1f}")
print(f"SMs used {len(np.unique(sm))}; rows per SM: max {np.bincount(sm).max()} min {np.bincount(sm)[np.unique(sm)].min()}")
# resident CTAs over time
grid = np.linspace(0, ge.max(), 40)
res = [(np.sum((gs <= x) & (ge > x))) for x in grid]
print("resident CTAs over time:", " ".join(f"{x:.0f}:{r}" for x, r in zip(grid, res)))
order = np.argsort(gs)
print("start-time quantiles us:", [round(float(np.percentile(gs, q)), 1) for q in (0, 25, 50, 60, 61, 70, 90, 100)])
# per SM: max concurrent
mc = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    ev = sorted([(gs[i], 1) for i in idx] + [(ge[i], -1) for i in idx])
    c = m = 0
    for _, d in ev:
        c += d; m = max(m, c)
    mc.append(m)
print("max concurrent CTAs per SM histogram:", np.bincount(mc))
slow = np.argsort(-ge)[:8]
print("last-finishing rows (row, layer, start, dur):", [(int(r), int(r % 61), round(float(gs[r]), 1), round(float(dur[r]), 1)) for r in slow])
_, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False)
st = st.cpu().numpy()
print("stats of the 8 longest rows:", gvr.STATS_FIELDS)
for r in np.argsort(-dur)[:8]:
    print(int(r), int(r % 61), round(float(dur[r]), 1), "stream cycles", int(t[r, 2] - t[r, 1]), "phase4", int(t[r, 4] - t[r, 3]),
          "out", int(t[r, 5] - t[r, 4]), list(st[r]))
