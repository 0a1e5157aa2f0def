"""Table-8 / Phase-2 replay analog on the cfg2 batch (PAPER.md:1088-1176,
576-586, 643-646, 1672-1683): per-kernel times of one call (CUDA events between the
kernels: guess = Phases 1-2, filter = the one HBM pass, refine = Phase 4 + ordered output),
the refine's per-row clock64 phases, and the Phase-2 statistics of every row — probes I
(distribution and CDF, by layer group L0-1 / L2-60 as in PAPER.md:576-586), exits,
candidates — with the kernel's T_c / I / exit checked row by row against the CPU replay
(oracle/phase2_replay.py).  Prints one JSON object."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from oracle import phase2_replay as P2
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
K = bench.K
F = gvr.STATS_FIELDS
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
R = b["R"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
kt = []
for i in range(8):
    flush.zero_()
    gvr.topk_events(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], events=evs)
    torch.cuda.synchronize()
    kt.append([evs[j].elapsed_time(evs[j + 1]) * 1e3 for j in range(3)])
kt = np.median(np.array(kt[2:]), axis=0)
_, ts = gvr.topk_phase_timing(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"])
_, _, st = gvr.topk_ex(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], values=False)
torch.cuda.synchronize()
t = ts.cpu().numpy().astype(np.int64)
st = st.cpu().numpy()
d = np.diff(t[t[:, 5] > 0][:, :6], axis=1)
I = st[:, F.index("secant_iters")]
layer = np.tile(np.arange(61), 8)  # rows are (request, layer)


def cdf(v):
    return {"I=1": round(float(np.mean(v <= 1)), 3), "I<=2": round(float(np.mean(v <= 2)), 3),
            "I<=3": round(float(np.mean(v <= 3)), 3), "I<=4": round(float(np.mean(v <= 4)), 3),
            "mean": round(float(v.mean()), 2), "max": int(v.max())}


# kernel vs replay, row by row (torch rows are 16-B aligned; N = 100,000 keeps every row aligned)
host = b["scores"].cpu().numpy()
prev = b["prev"].cpu().numpy()
agree = 0
for r in range(R):
    rep = P2.replay_row(host[r, :100_000], prev[r], K, head=0, filter_path=True)
    agree += int((rep["Tc"], rep["I"], rep["done"]) == (int(st[r, F.index("tc_key")]) & 0xFFFFFFFF, int(I[r]),
                                                        int(st[r, F.index("phase2_exit")])))
out = {
    "workload": "cfg2: 488 Eq.-1 decode rows, N = 100,000, K = 2048, previous-step guesses",
    "kernel_us_serialised": {"gvr_guess_kernel (Phases 1-2)": round(float(kt[0]), 1),
                             "gvr_filter_kernel (HBM pass)": round(float(kt[1]), 1),
                             "gvr_refine_kernel + gvr_fixup_kernel (Phase 4, output)": round(float(kt[2]), 1)},
    "refine_row_cycles_median": dict(zip(["records", "histogram", "kth_bin", "scatter", "rank_output"],
                                         [int(x) for x in np.median(d, axis=0)])),
    "phase2_I_all": cdf(I), "phase2_I_L0_1": cdf(I[layer < 2]), "phase2_I_L2_60": cdf(I[layer >= 2]),
    "phase2_I_hist": np.bincount(I, minlength=13).tolist(),
    "phase2_exits": dict(zip(gvr.PHASE2_EXITS.values(), np.bincount(st[:, F.index("phase2_exit")], minlength=4).tolist())),
    "candidates_per_row_mean": round(float(st[:, F.index("cand_count")].mean()), 1),
    "candidates_over_K": round(float(st[:, F.index("cand_count")].mean()) / K, 3),
    "replay_agreement_rows": f"{agree}/{R}",
    "paper_reference": "PAPER.md:576-586: I=1 67.6%, <=2/3/4 84.3/94.8/99.4%, max 6 (real logits, window [K, C])",
}
print(json.dumps(out, indent=1))
