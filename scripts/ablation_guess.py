"""Guess-source and distribution ablation (the paper's Table 9 /
Table 7 analog).

Part A — guess sources on the cfg2 batch (488 Eq.-1 decode rows, N = 100K): previous-step
Top-K (the method), static RoPE prior (Eq. 3), random positions, the adversarial lowest-K
positions, and no guess; GVR time per step and speedup over the radix baseline, with the
per-row statistics (passes, raises, candidates) and the measured overlap alpha of the
guess with the exact Top-K.

Part B — value distributions (synth.DISTRIBUTIONS shapes, N = 100K, 488 rows, random
guess): GVR vs radix time.

Every output is checked against the CPU oracle on a sample of rows.  Prints JSON lines."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, oracle, synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--dists", default="normal,lognormal,heavy_tail,uniform,few_distinct,negative")
args = ap.parse_args()
dev = torch.device("cuda:0")
K = bench.K


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / args.steps


def check(scores, lens, out, rows=(0, 1, 2, 100, 487)):
    host = scores.cpu().numpy()
    ln = lens.cpu().numpy()
    o = out.cpu().numpy()
    for r in rows:
        if r < host.shape[0]:
            assert np.array_equal(o[r], oracle.topk(host[r, :ln[r]], K)), f"row {r} differs from the oracle"


b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
scores, lens, R = b["scores"], b["row_lens"], b["R"]
host = scores.cpu().numpy()
exact = oracle.topk_batched(host, K, row_lens=lens.cpu().numpy())
radix_us = timeit(lambda: gvr.radix_topk(scores, K, row_lens=lens))
sources = {
    "prev_step": b["prev"],
    "static_prior": torch.from_numpy(np.stack([synth.guess("static", host[r], K, r) for r in range(R)]).astype(np.int32)).to(dev),
    "random": torch.from_numpy(np.stack([synth.guess("random", host[r], K, r) for r in range(R)]).astype(np.int32)).to(dev),
    "adversarial_lowest": torch.from_numpy(np.stack([synth.guess("adversarial", host[r], K, r) for r in range(R)]).astype(np.int32)).to(dev),
    "none": None,
}
for name, prev in sources.items():
    out = gvr.topk(scores, K, row_lens=lens, prev=prev)
    torch.cuda.synchronize()
    check(scores, lens, out)
    _, _, st = gvr.topk_ex(scores, K, row_lens=lens, prev=prev, values=False)
    st = st.cpu().numpy()
    us = timeit(lambda: gvr.topk(scores, K, row_lens=lens, prev=prev))
    alpha = None
    if prev is not None:
        pv = prev.cpu().numpy()
        alpha = float(np.mean([len(np.intersect1d(pv[r], exact[r])) / K for r in range(0, R, 4)]))
    print(json.dumps({"part": "A", "guess": name, "alpha": None if alpha is None else round(alpha, 3),
                      "gvr_us_per_step": round(us, 1), "radix_us_per_step": round(radix_us, 1),
                      "speedup": round(radix_us / us, 3), "passes_mean": float(st[:, 4].mean()),
                      "two_pass_rows": float(np.mean(st[:, 4] >= 2)), "raises_mean": float(st[:, 5].mean()),
                      "fallback_rows": float(np.mean(st[:, 3] >= 2)), "cand_mean": float(st[:, 2].mean())}), flush=True)

for dist in args.dists.split(","):
    rows = np.stack([synth.dist_row(dist, 100_000, seed=900 + r) for r in range(R)]).astype(np.float32)
    s = torch.from_numpy(rows).to(dev)
    ln = torch.full((R,), 100_000, dtype=torch.int32, device=dev)
    prev = torch.from_numpy(np.stack([synth.guess("random", rows[r], K, r) for r in range(R)]).astype(np.int32)).to(dev)
    out = gvr.topk(s, K, row_lens=ln, prev=prev)
    torch.cuda.synchronize()
    check(s, ln, out)
    us = timeit(lambda: gvr.topk(s, K, row_lens=ln, prev=prev))
    rus = timeit(lambda: gvr.radix_topk(s, K, row_lens=ln))
    _, _, st = gvr.topk_ex(s, K, row_lens=ln, prev=prev, values=False)
    st = st.cpu().numpy()
    print(json.dumps({"part": "B", "distribution": dist, "guess": "random", "gvr_us_per_step": round(us, 1),
                      "radix_us_per_step": round(rus, 1), "speedup": round(rus / us, 3),
                      "raises_mean": float(st[:, 5].mean()), "two_pass_rows": float(np.mean(st[:, 4] >= 2)),
                      "fallback_rows": float(np.mean(st[:, 3] >= 2))}), flush=True)
