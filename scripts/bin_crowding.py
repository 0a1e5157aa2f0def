"""Inspect the ordered-output binning of one row: T*, kmax and the occupancy of 2048
linear key bins over [T*, kmax] (the emit_sorted mapping)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--rows", default="247,431,435,100")
args = ap.parse_args()
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, args.batch))
def key(x):
    u = x.view(np.uint32).astype(np.uint64)
    return np.where(u >> 31 == 1, (~u) & 0xffffffff, u | 0x80000000).astype(np.uint64)
for r in [int(v) for v in args.rows.split(",")]:
    n = int(b["row_lens"][r])
    x = b["scores"][r, :n].cpu().numpy()
    k = key(x)
    ks = np.sort(k)[::-1]
    tstar, kmax = ks[2047], ks[0]
    sel = ks[:2048]
    d = sel - tstar
    rng = int(kmax - tstar) + 1
    bins = (d * 2048 // rng).astype(np.int64)
    cnt = np.bincount(bins, minlength=2048)
    xs = np.sort(x)[::-1]
    print(f"row {r} layer {r % 61}: top values {xs[:5]} ... K-th {xs[2047]:.4f}; key range {rng}; "
          f"max bin {cnt.max()} (bin {cnt.argmax()}), bins>32: {(cnt > 32).sum()}, nonempty {(cnt > 0).sum()}")
    print("   value quantiles of top-K:", np.round(np.percentile(xs[:2048], [0, 50, 90, 99, 99.9, 100]), 4))

# average in-bin rank-loop length (sum c^2 / n) of several bin mappings over the
# selected keys, on every 20th row of the batch
def loop_len(d, nb, f):
    b = np.minimum((f(d) * nb).astype(np.int64), nb - 1)
    c = np.bincount(b, minlength=nb)
    return float((c.astype(np.float64) ** 2).sum() / len(d)), int(c.max())
maps = {
    "linear2048": (2048, lambda d: d / (d.max() + 1)),
    "linear4096": (4096, lambda d: d / (d.max() + 1)),
    "sqrt2048": (2048, lambda d: np.sqrt(d / (d.max() + 1))),
    "log2048": (2048, lambda d: np.log2(1 + d) / np.log2(2 + d.max())),
    "rank-ideal": (2048, lambda d: (np.argsort(np.argsort(d)) / len(d))),
}
acc = {m: [] for m in maps}
for r in range(0, b["R"], 20):
    n = int(b["row_lens"][r])
    k = np.sort(key(b["scores"][r, :n].cpu().numpy()))[::-1][:2048]
    d = (k - k[-1]).astype(np.float64)
    for m, (nb, f) in maps.items():
        acc[m].append(loop_len(d, nb, f))
for m, v in acc.items():
    v = np.array(v)
    print(f"{m:12s} mean loop {v[:, 0].mean():6.2f}  worst row loop {v[:, 0].max():6.2f}  worst bin {v[:, 1].max():.0f}")
