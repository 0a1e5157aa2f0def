"""Filter-path CTA timeline on a bench config (gvr_cta_timeline): when each
persistent filter CTA starts, when its wait for Phases 1-2 ends and when it exits, to see
whether the spread of exit times comes from late starts or from uneven streaming."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
dev = torch.device("cuda:0")
b = bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.BASE_SEED, draft=cfg["draft"])
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for _ in range(3):
    gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
torch.cuda.synchronize()
for rep in range(2):
    flush.zero_()
    torch.cuda.synchronize()
    gvr.cta_timeline(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
    e1.record()
    t = gvr.cta_timeline(False, "filter")
    gt = gvr.cta_timeline(False, "guess")[:b["R"]]
    G = 3 * torch.cuda.get_device_properties(0).multi_processor_count
    t = t[:G]
    t0 = min(t[:, 0].min(), gt[:, 0].min())
    gs_, ge_ = (gt[:, 0] - t0) / 1e3, (gt[:, 1] - t0) / 1e3
    st, wt, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    q = lambda a: " ".join(f"{np.percentile(a, p):.1f}" for p in (0, 10, 50, 90, 100))
    print(f"call {e0.elapsed_time(e1) * 1e3:.1f} us; filter CTAs {G}; times from the first guess CTA start (us), p0/10/50/90/100")
    print("  guess start", q(gs_))
    print("  guess end  ", q(ge_))
    print("  guess dur  ", q(ge_ - gs_))
    gl_, gp1_ = (gt[:, 2] - t0) / 1e3, (gt[:, 3] - t0) / 1e3
    print("  guess loads", q(gl_), " phase1 done", q(gp1_), " phase2 dur", q(ge_ - gp1_))
    print("  start      ", q(st))
    print("  wait end   ", q(wt))
    print("  exit       ", q(en))
    print("  stream dur ", q(en - wt))
    print("  corr(start, exit) %.2f  corr(wait end, exit) %.2f" % (np.corrcoef(st, en)[0, 1], np.corrcoef(wt, en)[0, 1]))
    sm = t[:, 3]
    per_sm = np.array([en[sm == s].max() for s in np.unique(sm)])
    print("  per-SM last exit", q(per_sm), " CTA index vs exit corr %.2f" % np.corrcoef(np.arange(G), en)[0, 1])
    # exit time by CTA index decile
    print("  exit by CTA-index decile:", " ".join(f"{en[i * G // 10:(i + 1) * G // 10].mean():.1f}" for i in range(10)))
