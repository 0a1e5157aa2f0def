import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench, synth
import paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
rho = 0.95
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, 77, int(rho * 1000)), rho=rho)
for _ in range(3):
    out, _, st = gvr.radix2_topk_ex(b["scores"], bench.K, row_lens=b["row_lens"]) if hasattr(gvr, "radix2_topk_ex") else (None, None, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): gvr.radix2_topk(b["scores"], bench.K, row_lens=b["row_lens"])
e1.record(); torch.cuda.synchronize()
print("radix2 us", e0.elapsed_time(e1) * 1e3 / 5)
if st is not None:
    st = st.cpu().numpy(); F = gvr.STATS_FIELDS
    print("raises", np.bincount(st[:, F.index("raises")]), "snap>0", (st[:, 1] > 0).sum(), "cand max", st[:, 2].max(), "done", np.bincount(st[:, 3]))
    slow = np.argsort(-st[:, 2])[:3]
    for r in slow: print(r, dict(zip(F, st[r].tolist())))
