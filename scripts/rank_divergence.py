"""Model of select_sorted's in-bin rank loop on cfg2 rows: entries (top K of the ~f(T_c)
candidates) binned linearly over [T, kmax]; per warp of 32 consecutive sorted entries the
loop runs max(bin size) iterations.  Reports mean per-warp max for several bin counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
def key(x):
    u = x.view(np.uint32).astype(np.uint64)
    return np.where(u >> 31 == 1, (~u) & 0xffffffff, u | 0x80000000).astype(np.uint64)
res = {}
for r in range(2, b["R"], 9):
    n = int(b["row_lens"][r])
    k = np.sort(key(b["scores"][r, :n].cpu().numpy()))[::-1]
    cand = k[:3800]
    T, kmax = cand[-1], cand[0]
    for nb in (2048, 4096, 8192):
        scale = (nb << 32) // (int(kmax - T) + 1)
        bins = (nb - 1) - np.minimum(((cand - T).astype(np.uint64) * np.uint64(scale)) >> np.uint64(32), nb - 1).astype(np.int64)
        c = np.bincount(bins, minlength=nb)
        sel = np.sort(bins)[:2048]           # sorted positions 0..2047 in bin order
        per_entry = c[sel]
        warp_max = per_entry.reshape(64, 32).max(axis=1)
        res.setdefault(nb, []).append((per_entry.mean(), warp_max.mean()))
for nb, v in res.items():
    v = np.array(v)
    print(f"{nb} bins: mean loop {v[:, 0].mean():.2f}, mean per-warp max {v[:, 1].mean():.2f}")
