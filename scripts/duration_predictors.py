"""Which per-row quantities predict a row's duration in the streaming kernel (cfg2)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
for bi in range(2):
    b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, bi))
    for _ in range(3):
        out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
    _, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False)
    torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64); st = st.cpu().numpy()
    dur = (t[:, 7] - t[:, 6]) / 1e3
    stream = (t[:, 2] - t[:, 1]) / 1.965e3
    F = gvr.STATS_FIELDS
    light = st[:, F.index("raises")] == 0
    print(f"batch {bi}: rows {len(dur)}, light rows {light.sum()}, dur light p10/50/90 "
          f"{np.percentile(dur[light], 10):.1f}/{np.median(dur[light]):.1f}/{np.percentile(dur[light], 90):.1f} us")
    for name in ("buffer_count", "cand_count", "raises", "snap_iters"):
        v = st[:, F.index(name)].astype(float)
        cc = np.corrcoef(v[light], dur[light])[0, 1] if v[light].std() > 0 else float("nan")
        print(f"   corr(duration, {name}) on light rows: {cc:+.2f}")
    cs = np.corrcoef(stream[light], dur[light])[0, 1]
    print(f"   corr(duration, stream time): {cs:+.2f}; start-time corr {np.corrcoef((t[light, 6] - t[:, 6].min()), dur[light])[0, 1]:+.2f}")
