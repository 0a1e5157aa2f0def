import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch, bench, synth
import paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
for cname in ("cfg2", "cfg4"):
    cfg = bench.CONFIGS[cname]
    b = bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.BASE_SEED, draft=cfg["draft"])
    _, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False)
    st = st.cpu().numpy()
    print(cname, "narrowings per row:", np.bincount(st[:, 5]).tolist(), "cand p50/p90", np.percentile(st[:, 2], 50), np.percentile(st[:, 2], 90))
