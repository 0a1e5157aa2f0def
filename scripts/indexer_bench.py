"""Fused indexer -> Top-K vs the unfused path on an MTP-shaped decode batch:
R = requests x layers x drafts rows of N keys, the draft rows of a (request, layer) sharing
one bf16 key set (RoPE'd, from the Eq.-1 generator).  Times (CUDA events, 10 calls after 3
warm-ups): the indexer scores alone (gvr_indexer_scores), the unfused path (scores
materialised in HBM, then gvr_topk_batched) and the fused path (gvr_indexer_topk_batched);
checks fused == unfused bit for bit.  Prints one JSON object."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=4)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--drafts", type=int, default=4)
ap.add_argument("--n", type=int, default=100_000)
a = ap.parse_args()
dev = torch.device("cuda:0")
K = 2048
keys, qs, ws, rs = [], [], [], []
for si in range(a.requests * a.layers):
    lay = synth.IndexerLayer(a.n, synth.layer_rho(2 + si % 59, synth.BASE_SEED), synth.splitmix64(4000, si), dev)
    keys.append(lay.keys[:a.n].to(torch.bfloat16))
    for j in range(a.drafts):
        if j:
            lay.step()
        qs.append(lay.query(a.n).to(torch.bfloat16))
        ws.append(lay.w.clone())
        rs.append(si)
    del lay
keys = torch.stack(keys).contiguous()
q = torch.stack(qs).contiguous()
w = torch.stack(ws).float().contiguous()
row_set = torch.tensor(rs, dtype=torch.int32, device=dev)
R = row_set.shape[0]
lens = torch.full((R,), a.n, dtype=torch.int32, device=dev)
sc = torch.empty((R, a.n), dtype=torch.float32, device=dev)
prev = gvr.topk(gvr.indexer_scores(keys, row_set, q, w), K)  # a guess: this step's own Top-K shifted by noise-free
prev = torch.roll(prev, 1, dims=0).contiguous()               # ... of a neighbouring row (alpha ~ layer overlap)
out_f = torch.empty((R, K), dtype=torch.int32, device=dev)
out_u = torch.empty((R, K), dtype=torch.int32, device=dev)


def t(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


t_sc = t(lambda: gvr.indexer_scores(keys, row_set, q, w, row_lens=lens, out=sc))
t_un = t(lambda: (gvr.indexer_scores(keys, row_set, q, w, row_lens=lens, out=sc),
                  gvr.topk(sc, K, row_lens=lens, prev=prev, out=out_u)))
t_fu = t(lambda: gvr.indexer_topk(keys, row_set, q, w, K, row_lens=lens, prev=prev, out=out_f, scratch=sc))
torch.cuda.synchronize()
same = bool(torch.equal(out_f, out_u))
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
key_bytes = R * a.n * 256  # every row streams its key set (draft rows read it separately)
flops = R * a.n * 64 * 128 * 2
print(json.dumps({
    "workload": f"{a.requests} requests x {a.layers} layers x {a.drafts} drafts = {R} rows, N = {a.n}, 64 heads x 128 (bf16)",
    "indexer_scores_us": round(t_sc, 1), "unfused_us": round(t_un, 1), "fused_us": round(t_fu, 1),
    "fused_speedup_vs_unfused": round(t_un / t_fu, 3), "fused_equals_unfused": same,
    "fused_key_gbs": round(key_bytes / (t_fu * 1e-6) / 1e9, 1),
    "fused_hbm_frac": round(key_bytes / (t_fu * 1e-6) / 1e9 / peaks["hbm_gbs"], 3),
    "fused_tflops": round(flops / (t_fu * 1e-6) / 1e12, 1),
    "scores_tflops": round(flops / (t_sc * 1e-6) / 1e12, 1),
    "score_row_bytes_saved_per_call": int(2 * R * a.n * 4),
}, indent=1))
