"""Which rows of a cfg2 batch are slow in the streaming pass, and why (stats per row)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
for _ in range(3):
    out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
_, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False)
torch.cuda.synchronize()
t = ts.cpu().numpy().astype(np.int64); st = st.cpu().numpy()
stream = t[:, 2] - t[:, 1]
F = gvr.STATS_FIELDS
order = np.argsort(-stream)
print("row layer stream_cycles total_cycles", " ".join(F))
for r in order[:20]:
    print(r, r % 61, stream[r], t[r, 5] - t[r, 0], " ".join(str(x) for x in st[r]))
print("raises by layer (mean):", {l: float(st[np.arange(len(st)) % 61 == l, F.index("raises")].mean()) for l in range(4)})
