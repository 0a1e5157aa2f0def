# pathological refine rows: the dense part of the list is negative, a few outliers far above
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle, paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
K = 2048
R, n = 488, 100_000
rng = np.random.default_rng(5)
host = (-1.0 + 1e-3 * rng.standard_normal((R, n))).astype(np.float32)   # dense negatives
for r in range(R):
    pos = rng.choice(n, 12, replace=False)
    host[r, pos] = (100.0 + 50 * rng.random(12)).astype(np.float32)       # far positive outliers
s = torch.from_numpy(host).to(dev)
lens = torch.full((R,), n, dtype=torch.int32, device=dev)
for _ in range(3):
    out, _, st = gvr.topk_ex(s, K, row_lens=lens, values=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    gvr.topk(s, K, row_lens=lens)
e1.record(); torch.cuda.synchronize()
print("us per call", e0.elapsed_time(e1) * 1e3 / 5)
ref = oracle.topk_batched(host, K)
print("exact", np.array_equal(out.cpu().numpy(), ref))
st = st.cpu().numpy()
print("cand mean", st[:, 2].mean(), "raises", np.bincount(st[:, 5]), "snap>0 (fixup rows)", (st[:, 1] > 0).sum())
