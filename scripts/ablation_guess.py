"""Guess-source, distribution and alpha ablation on the default batch (filter) path
(the paper's Table 9 / Table 7 analogs, PAPER.md:1029-1086,
965-1027).  488-row batches of N = 100K, GVR vs both radix baselines (radix: one CTA per
row; radix2: the same-geometry radix), CUDA events over 20 rotated calls, plus per-row
statistics: the guess's overlap alpha with the exact Top-K, Phase-2 probes I (mean and
histogram), candidates, passes and done kinds.  Every output is checked against the CPU
oracle on sampled rows.  Prints one JSON line per case.

Part A — guess sources on the cfg2 batch (Eq.-1 decode rows): previous-step Top-K (the
method), the static RoPE prior (Eq. 3), random positions, the adversarial lowest-K
positions, no guess.
Part B — the Table-7 score shapes (beta, weibull, logistic, lognormal) with a correlated
previous step (the Top-K of the row plus 0.3 sd of noise: alpha ~0.4-0.5), and App.-E
synthetic rows (N = 70,690) with the static prior.
Part C — alpha sweep: Eq.-1 batches with every layer's AR coefficient rho fixed."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, oracle, synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--parts", default="A,B,C")
args = ap.parse_args()
dev = torch.device("cuda:0")
K = bench.K
F = gvr.STATS_FIELDS


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


def run_case(tag, scores, lens, prev, exact=None, **extra):
    out = gvr.topk(scores, K, row_lens=lens, prev=prev)
    torch.cuda.synchronize()
    host = scores.cpu().numpy()
    ln = lens.cpu().numpy()
    o = out.cpu().numpy()
    for r in (0, 1, 2, 100, scores.shape[0] - 1):
        assert np.array_equal(o[r], oracle.topk(host[r, :ln[r]], K)), f"{tag}: row {r} differs from the oracle"
    us = timeit(lambda: gvr.topk(scores, K, row_lens=lens, prev=prev))
    rus = timeit(lambda: gvr.radix_topk(scores, K, row_lens=lens))
    r2us = timeit(lambda: gvr.radix2_topk(scores, K, row_lens=lens))
    _, _, st = gvr.topk_ex(scores, K, row_lens=lens, prev=prev, values=False)
    st = st.cpu().numpy()
    alpha = None
    if prev is not None:
        if exact is None:
            exact = oracle.topk_batched(host[::8], K, row_lens=ln[::8])
            pv = prev.cpu().numpy()[::8]
        else:
            pv = prev.cpu().numpy()
        alpha = float(np.mean([len(np.intersect1d(pv[r], exact[r])) / K for r in range(len(pv))]))
    I = st[:, F.index("secant_iters")]
    rec = {"case": tag, **extra, "alpha": None if alpha is None else round(alpha, 3),
           "gvr_us_per_step": round(us, 1), "radix_us_per_step": round(rus, 1), "radix2_us_per_step": round(r2us, 1),
           "speedup_vs_radix": round(rus / us, 3), "speedup_vs_radix2": round(r2us / us, 3),
           "phase2_I_mean": round(float(I.mean()), 2), "phase2_I_hist": np.bincount(I, minlength=13).tolist(),
           "phase2_exits": np.bincount(st[:, F.index("phase2_exit")], minlength=4).tolist(),
           "cand_mean": round(float(st[:, F.index("cand_count")].mean()), 1),
           "passes_mean": round(float(st[:, F.index("global_passes")].mean()), 3),
           "done_kinds": np.bincount(st[:, F.index("done_kind")], minlength=4).tolist()}
    print(json.dumps(rec), flush=True)


parts = args.parts.split(",")
if "A" in parts:
    b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
    scores, lens, R = b["scores"], b["row_lens"], b["R"]
    host = scores.cpu().numpy()
    sources = {
        "prev_step": b["prev"],
        "static_prior": torch.from_numpy(np.stack([synth.guess("static", host[r], K, r) for r in range(R)])).to(dev),
        "random": torch.from_numpy(np.stack([synth.guess("random", host[r], K, r) for r in range(R)])).to(dev),
        "adversarial_lowest": torch.from_numpy(np.stack([synth.guess("adversarial", host[r], K, r)
                                                         for r in range(R)])).to(dev),
        "none": None,
    }
    for name, prev in sources.items():
        run_case("A", scores, lens, prev, guess=name, workload="cfg2 Eq.-1 decode rows")

if "B" in parts:
    R, N = 488, 100_000
    for dist in synth.TABLE7_SHAPES:
        rows = np.stack([synth.dist_row(dist, N, seed=900 + r) for r in range(R)]).astype(np.float32)
        rng = np.random.default_rng(901)
        prevrows = rows + (0.3 * rows.std(axis=1, keepdims=True) * rng.standard_normal(rows.shape)).astype(np.float32)
        prev = torch.from_numpy(oracle.topk_batched(prevrows, K)).to(dev)
        run_case("B", torch.from_numpy(rows).to(dev), torch.full((R,), N, dtype=torch.int32, device=dev), prev,
                 distribution=dist, guess="correlated previous step (0.3 sd noise)")
    n = 70_690
    rows = np.stack([synth.appendix_e_row(n, seed=950 + r).numpy() for r in range(R)]).astype(np.float32)
    prior = synth.static_prior(n, K, query_pos=0)
    prev = torch.from_numpy(np.tile(prior, (R, 1))).to(dev)
    run_case("B", torch.from_numpy(rows).to(dev), torch.full((R,), n, dtype=torch.int32, device=dev), prev,
             distribution="appendix_e (N=70,690)", guess="static RoPE prior (Eq. 3)")

if "C" in parts:
    for rho in (0.0, 0.5, 0.8, 0.9, 0.95, 0.98, 0.995):
        b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, 77, int(rho * 1000)),
                                    rho=rho)
        run_case("C", b["scores"], b["row_lens"], b["prev"], rho=rho, guess="prev_step")
