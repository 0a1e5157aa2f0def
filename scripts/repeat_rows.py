"""Run the same batch several times; per-phase cycles of selected rows each time
(determinism check of per-row costs)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2604_22312_b200 as gvr
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--rows", default="247,431,435")
ap.add_argument("--reps", type=int, default=4)
args = ap.parse_args()
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.splitmix64(synth.BASE_SEED, args.batch))
rows = [int(v) for v in args.rows.split(",")]
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for rep in range(args.reps):
    flush.zero_()
    out, ts = gvr.topk_phase_timing(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"])
    torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64)
    d = np.diff(t[:, :6], axis=1)
    worst = np.argsort(-d[:, 4])[:3]
    print(f"rep {rep}: rows {rows} out-cycles {[int(d[r, 4]) for r in rows]} phase4 {[int(d[r, 3]) for r in rows]}; "
          f"worst out rows {[(int(r), int(d[r, 4]), int(t[r, 8])) for r in worst]}")
