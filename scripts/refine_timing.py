"""Batch filter path on a bench config: per-row clock64 phases of gvr_refine_kernel (pop ->
segment records -> histogram pass -> K-th bin -> scatter -> rank/output) and the refine CTA
timeline (globaltimer), plus the four kernels' CUDA-event times (serialised)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr

dev = torch.device("cuda:0")
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
b = bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.BASE_SEED, draft=cfg["draft"])
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for _ in range(3):
    out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
torch.cuda.synchronize()
flush.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
e1.record()
torch.cuda.synchronize()
print(f"whole call (PDL, phase stamps on): {e0.elapsed_time(e1) * 1e3:.1f} us")
t = ts.cpu().numpy().astype(np.int64)
ok = t[:, 5] > 0
print(f"rows refined from lists: {ok.sum()} of {len(t)}")
t = t[ok]
gs, ge = t[:, 6], t[:, 7]
t0 = gs.min()
gs, ge = (gs - t0) / 1e3, (ge - t0) / 1e3
dur = ge - gs
print(f"refine rows span {ge.max():.1f} us after the first pop; duration p10/50/90/max "
      f"{np.percentile(dur,10):.1f}/{np.median(dur):.1f}/{np.percentile(dur,90):.1f}/{dur.max():.1f} us")
names = ["records", "hist_pass", "kth_bin", "scatter", "rank_out"]
d = np.diff(t[:, :6], axis=1)
for i, nm in enumerate(names):
    print(f"{nm:10s} cycles median {np.median(d[:, i]):8.0f} p90 {np.percentile(d[:, i], 90):8.0f} max {d[:, i].max():8.0f}")
grid = np.linspace(0, ge.max(), 25)
print("busy refine CTAs:", " ".join(f"{x:.0f}:{np.sum((gs <= x) & (ge > x))}" for x in grid))
print("pop times (us) p10/50/90/max:", [round(float(np.percentile(gs, q)), 1) for q in (10, 50, 90, 100)])
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(5):
    flush.zero_()
    gvr.topk_events(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], events=evs)
torch.cuda.synchronize()
print("serialised events us: guess %.1f filter %.1f refine+fixup %.1f" % tuple(evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(3)))
for _ in range(3):
    flush.zero_()
    e0.record()
    gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
    e1.record()
torch.cuda.synchronize()
print(f"whole call (PDL): {e0.elapsed_time(e1) * 1e3:.1f} us")
_, _, st = gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], values=False)
st = st.cpu().numpy()
tt = ts.cpu().numpy().astype(np.int64)
okr = np.nonzero(tt[:, 5] > 0)[0]
durr = (tt[okr, 7] - tt[okr, 6]) / 1e3
for j in np.argsort(-durr)[:5]:
    r = int(okr[j])
    print("slow row", r, f"{durr[j]:.1f} us", "stats", st[r].tolist(), "phases", np.diff(tt[r, :6]).tolist(), "sm", int(tt[r, 8]))
