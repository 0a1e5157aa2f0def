"""Per-phase clock64 breakdown of the GVR kernel (Table 8 analog).
Runs the cfg2 batch (488 rows, 2 CTAs/SM contention) and a batch-1 row (CTA alone)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
res = {}
for name, (req, lay, n) in {"cfg2_batch488": (8, 61, 100_000), "batch1_N100K": (1, 3, 100_000)}.items():
    b = bench.make_decode_batch(req, lay, n, dev, seed=synth.BASE_SEED)
    sel = slice(None) if req > 1 else slice(2, 3)  # batch-1: one correlated-layer row
    scores, lens, prev = b["scores"][sel].contiguous(), b["row_lens"][sel].contiguous(), b["prev"][sel].contiguous()
    for _ in range(3):
        out, ts = gvr.topk_phase_timing(scores, bench.K, row_lens=lens, prev=prev)
    torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64)
    ok = (t[:, 1:6] > 0).all(axis=1)
    d = np.diff(t[ok, :6], axis=1)
    tot = t[ok, 5] - t[ok, 0]
    row = {"rows": int(ok.sum()), "total_cycles_median": float(np.median(tot)),
           "total_cycles_p10_p90_p99_max": [float(np.percentile(tot, q)) for q in (10, 90, 99, 100)],
           "stream_p90_p99_max": [float(np.percentile(d[:, 1], q)) for q in (90, 99, 100)]}
    for i, ph in enumerate(gvr.PHASES):
        row[ph] = {"median": float(np.median(d[:, i])), "mean": float(d[:, i].mean()),
                   "share": float(d[:, i].sum() / tot.sum())}
    res[name] = row
    print(name, json.dumps(row, indent=None))
