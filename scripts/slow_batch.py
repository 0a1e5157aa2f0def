"""Why is one batch slow?  Per-row stats and refine phase stamps of a decode batch with a
given AR coefficient (ablation part C): rows sent to the fixup, narrowing levels, the
slowest refine rows and the kernel times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
rho = float(sys.argv[1]) if len(sys.argv) > 1 else 0.98
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, 77, int(rho * 1000)), rho=rho)
K = bench.K
_, _, st = gvr.topk_ex(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], values=False)
st = st.cpu().numpy()
F = gvr.STATS_FIELDS
print("done_kind counts", np.bincount(st[:, F.index("done_kind")], minlength=4), "raises", np.bincount(st[:, F.index("raises")]),
      "cluster field", np.bincount(st[:, F.index("cluster")]))
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(3):
    gvr.topk_events(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], events=evs)
torch.cuda.synchronize()
print("serialised events us: guess %.1f filter %.1f refine+fixup %.1f" % tuple(evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(3)))
out, ts = gvr.topk_phase_timing(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"])
torch.cuda.synchronize()
t = ts.cpu().numpy().astype(np.int64)
ok = t[:, 5] > 0
print("rows with refine stamps", ok.sum(), "of", len(t), "; rows without:", np.nonzero(~ok)[0][:20].tolist())
d = (t[ok, 7] - t[ok, 6]) / 1e3
order = np.argsort(-d)[:6]
rows = np.nonzero(ok)[0]
for j in order:
    r = rows[j]
    print("row", r, f"{d[j]:.1f} us", dict(zip(F, st[r].tolist())), "phases", np.diff(t[r, :6]).tolist())
for r in np.nonzero(~ok)[0][:5]:
    print("unstamped row", r, dict(zip(F, st[r].tolist())))
