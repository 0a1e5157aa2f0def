"""Calibrate the collect-threshold width per row length: for each N, 8 decode rows of
correlated layers (rho ~ 0.9) with their previous-step guesses; per sigma: fraction of
rows needing the second pass (f(T_c) < K), raises per row, and time of the 8-row batch."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="8192,16384,32768,65536,131072")
ap.add_argument("--sigmas", default="0.3,0.5,0.7,1.0")
ap.add_argument("--rows", type=int, default=8)
args = ap.parse_args()
dev = torch.device("cuda:0")
K = bench.K
for n in [int(x) for x in args.ns.split(",")]:
    b = bench.make_decode_batch(args.rows, 1, n, dev, seed=synth.splitmix64(synth.BASE_SEED, n), first_layer=30)
    for sg in [float(x) for x in args.sigmas.split(",")]:
        opt = gvr.GvrOptions(sg, 0, 0, 0)
        _, _, st = gvr.topk_ex(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], values=False, options=opt)
        st = st.cpu().numpy()
        for _ in range(3):
            gvr.topk_ex(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], values=False, stats=False, options=opt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            gvr.topk_ex(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], values=False, stats=False, options=opt)
        e1.record()
        torch.cuda.synchronize()
        print(f"N {n:6d} sigma {sg:4.2f}: {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us/batch  two-pass {np.mean(st[:, 4] >= 2):.2f}"
              f"  raises {st[:, 5].mean():.2f}  f(Tc) {st[:, 6].mean():.0f}  cluster {st[0, 7]}", flush=True)
