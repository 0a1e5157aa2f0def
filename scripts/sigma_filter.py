"""Collect-threshold width sigma (R22) on the batch filter path: call time, mean
list length and fallback rows (global passes > 1) for cfg2 / cfg4 over 3 batches each."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for cname in ("cfg2", "cfg4"):
    cfg = bench.CONFIGS[cname]
    batches = [bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev,
                                       seed=synth.splitmix64(synth.BASE_SEED, b), draft=cfg["draft"]) for b in range(3)]
    for sigma in (0.3, 0.25, 0.2, 0.15):
        opt = gvr.GvrOptions(sigma, 0, 0, 0, 0)
        ts, cand, fall = [], [], 0
        for rep in range(4):
            for b in batches:
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], options=opt)
                e1.record()
                torch.cuda.synchronize()
                if rep > 0:
                    ts.append(e0.elapsed_time(e1) * 1e3)
        for b in batches:
            _, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False, options=opt)
            st = st.cpu().numpy()
            cand.append(st[:, 2].mean())
            fall += int((st[:, 4] > 1).sum())
        print(json.dumps({"config": cname, "sigma": sigma, "us_median": round(float(np.median(ts)), 1),
                          "cand_mean": round(float(np.mean(cand)), 1), "fallback_rows": fall,
                          "rows": 3 * batches[0]["R"]}), flush=True)
