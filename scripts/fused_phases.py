"""Batch-1 (fused / cluster kernel) per-phase clock64 stamps of one decode row per N:
start -> Phases 1-2 done -> stream done -> Phase 3 -> Phase 4 -> end (cycles), plus the
Phase-2 probes I, and the CUDA-event latency of the call with L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
K = bench.K
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,32768,131072").split(",")]:
    lay = synth.IndexerLayer(n, synth.layer_rho(30, synth.BASE_SEED), synth.splitmix64(synth.BASE_SEED, n), dev)
    pr = lay.scores(n - 1)
    lay.step()
    row = lay.scores(n)[None, :].contiguous()
    ps = torch.zeros((1, n), dtype=torch.float32, device=dev)
    ps[0, :n - 1] = pr
    prev = gvr.topk(ps, K, row_lens=torch.tensor([n - 1], dtype=torch.int32, device=dev))
    stamps = []
    for _ in range(12):
        flush.zero_()
        _, ts = gvr.topk_phase_timing(row, K, prev=prev)
        torch.cuda.synchronize()
        stamps.append(ts.cpu().numpy()[0])
    t = np.array(stamps[2:], dtype=np.int64)
    d = np.diff(t[:, :6], axis=1)
    med = np.median(d, axis=0)
    lat = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gvr.topk(row, K, prev=prev)
        e1.record()
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    _, _, st = gvr.topk_ex(row, K, prev=prev, values=False)
    s = dict(zip(gvr.STATS_FIELDS, st.cpu().numpy()[0].tolist()))
    print(f"N={n}: event latency median {np.median(lat):.1f} us; cycles phase12 {med[0]:.0f} stream {med[1]:.0f} "
          f"phase3 {med[2]:.0f} phase4 {med[3]:.0f} output {med[4]:.0f} (total {med.sum():.0f}, "
          f"{(t[:, 7] - t[:, 6]).mean() / 1e3:.1f} us wall in-kernel); I={s['secant_iters']} cluster={s['cluster']} "
          f"cand={s['cand_count']}", flush=True)
