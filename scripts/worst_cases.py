"""Worst cases on the default batch path: 488-row batches of N = 100K
whose rows are all-equal, few-distinct, 90%-tied, with adversarial (lowest-K) or random
guesses, and very high alpha (rho 0.98) — GVR vs the radix baselines (one-CTA-per-row
radix and the same-geometry radix2), CUDA events, inputs rotated over 3 batches > L2.
Also the per-row passes / done kinds.  One JSON line per case."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, oracle, synth
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
K, R, N = bench.K, 488, 100_000


def timed(fn, batches, steps=10):
    for i in range(3):
        fn(batches[i % 3])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        fn(batches[i % 3])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


def dist_batch(kind, guess_kind, seed):
    host = np.stack([synth.dist_row(kind, N, seed=seed + r) for r in range(R)]).astype(np.float32)
    s = torch.from_numpy(host).to(dev)
    if guess_kind == "adversarial":
        prev = torch.argsort(s, dim=1, stable=True)[:, :K].to(torch.int32).contiguous()
    else:
        prev = torch.randint(0, N, (R, K), dtype=torch.int32, device=dev, generator=torch.Generator(dev).manual_seed(seed))
    return {"scores": s, "row_lens": torch.full((R,), N, dtype=torch.int32, device=dev), "prev": prev}


cases = [("all_equal", "random"), ("few_distinct", "random"), ("ties90", "random"), ("normal", "adversarial"),
         ("normal", "random"), ("lognormal", "adversarial")]
for kind, gk in cases + [("decode_rho0.98", "prev"), ("decode_rho0.0", "prev")]:
    if kind.startswith("decode"):
        rho = float(kind.split("rho")[1])
        bs = [bench.make_decode_batch(8, 61, N, dev, seed=synth.splitmix64(9100, i), rho=rho) for i in range(3)]
    else:
        bs = [dist_batch(kind, gk, 9000 + 1000 * i) for i in range(3)]
    for b in bs:
        b["out"] = torch.empty((R, K), dtype=torch.int32, device=dev)
    t_g = timed(lambda b: gvr.topk(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], out=b["out"]), bs)
    t_r = timed(lambda b: gvr.radix_topk(b["scores"], K, row_lens=b["row_lens"], out=b["out"]), bs)
    t_r2 = timed(lambda b: gvr.radix2_topk(b["scores"], K, row_lens=b["row_lens"], out=b["out"]), bs)
    idx, _, st = gvr.topk_ex(bs[0]["scores"], K, row_lens=bs[0]["row_lens"], prev=bs[0]["prev"], values=False)
    torch.cuda.synchronize()
    ok = bool(np.array_equal(idx.cpu().numpy(), oracle.topk_batched(bs[0]["scores"].cpu().numpy(), K)))
    st = st.cpu().numpy()
    print(json.dumps({"case": kind, "guess": gk, "gvr_us": round(t_g, 1), "radix_us": round(t_r, 1),
                      "radix2_us": round(t_r2, 1), "speedup_vs_radix": round(t_r / t_g, 3),
                      "speedup_vs_radix2": round(t_r2 / t_g, 3), "exact": ok,
                      "passes_mean": float(st[:, 4].mean()), "passes_max": int(st[:, 4].max()),
                      "fixup_rows": int((st[:, 4] > 1).sum()), "tiefill_rows": int((st[:, 3] == 2).sum()),
                      "phase2_I_mean": float(st[:, 0].mean()), "cand_mean": float(st[:, 2].mean())}), flush=True)
