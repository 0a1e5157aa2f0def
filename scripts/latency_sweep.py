"""Batch-1 latency sweep (cfg1 / cfg3; the paper's Table 5 analog):
one decode row at N = 8K ... 256K with its previous-step guess, GVR vs the radix
baseline, L2 flushed before every launch, CUDA events
around each launch, median / p10 / p90 over repetitions.  Also reports the per-row
stats (passes, raises, candidates).  Prints one JSON object per N."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="8192,16384,32768,65536,100000,131072,262144")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--layer", type=int, default=30, help="layer index (rho ~ 0.9 for layers >= 2)")
args = ap.parse_args()
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # 256 MB > 2 x L2
K = bench.K
for n in [int(x) for x in args.ns.split(",")]:
    lay = synth.IndexerLayer(n, synth.layer_rho(args.layer, synth.BASE_SEED), synth.splitmix64(synth.BASE_SEED, n), dev)
    prev_row = lay.scores(n - 1)
    lay.step()
    row = lay.scores(n)
    scores = row[None, :].contiguous()
    pscores = torch.zeros((1, n), dtype=torch.float32, device=dev)
    pscores[0, :n - 1] = prev_row
    prev = gvr.topk(pscores, K, row_lens=torch.tensor([n - 1], dtype=torch.int32, device=dev))
    lens = torch.tensor([n], dtype=torch.int32, device=dev)
    out = torch.empty((1, K), dtype=torch.int32, device=dev)
    res = {"N": n}
    for impl in ("gvr", "radix"):
        def call():
            if impl == "gvr":
                gvr.topk(scores, K, row_lens=lens, prev=prev, out=out)
            else:
                gvr.radix_topk(scores, K, row_lens=lens, out=out)
        for _ in range(3):
            call()
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts = np.array(ts)
        res[impl] = {"us_median": round(float(np.median(ts)), 2), "us_p10": round(float(np.percentile(ts, 10)), 2),
                     "us_p90": round(float(np.percentile(ts, 90)), 2)}
    _, _, st = gvr.topk_ex(scores, K, row_lens=lens, prev=prev, values=False)
    s = st.cpu().numpy()[0]
    res["speedup"] = round(res["radix"]["us_median"] / res["gvr"]["us_median"], 3)
    res["gvr_stats"] = dict(zip(gvr.STATS_FIELDS, [int(v) for v in s]))
    res["gvr_row_gbs"] = round(4 * n / (res["gvr"]["us_median"] * 1e-6) / 1e9, 1)
    print(json.dumps(res), flush=True)
