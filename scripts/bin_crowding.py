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
