#!/usr/bin/env python
"""CPU model of the batch path's Phase 1-2 (oracle/phase2_replay.py) on synthetic Eq.-1
decode rows: distribution of I (secant_iters), the Phase-2 exit kind and f(T_c)/K over
layers / rho values, for calibrating the window (R35).

    python scripts/phase2_model.py [--n 100000] [--requests 1] [--rhos 0.95,0.98,0.995]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from oracle import phase2_replay as P2  # noqa: E402
import synth  # noqa: E402

K = 2048


def rows(n, requests, layers, rhos, seed=synth.BASE_SEED, draft=1):
    for q in range(requests):
        for l in layers:
            rho = synth.layer_rho(l, seed) if rhos is None else rhos[l % len(rhos)]
            lay = synth.IndexerLayer(n + draft - 1, rho, synth.splitmix64(seed, 0, q, l))
            prev = lay.scores(n - 1).numpy()
            lay.step()
            for j in range(draft):
                if j:
                    lay.step()
                yield l, rho, j, prev, lay.scores(n + j).numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--requests", type=int, default=1)
    ap.add_argument("--layers", default="0-60")
    ap.add_argument("--rhos", default=None)
    ap.add_argument("--draft", type=int, default=1)
    ap.add_argument("--stride", type=int, default=8)  # guess stride (every row)
    a = ap.parse_args()
    lo, hi = (int(v) for v in a.layers.split("-"))
    rhos = [float(v) for v in a.rhos.split(",")] if a.rhos else None
    recs = []
    for l, rho, j, prev, cur in rows(a.n, a.requests, range(lo, hi + 1), rhos, draft=a.draft):
        g = oracle.topk(prev, K)
        top = oracle.topk(cur, K)
        alpha = len(np.intersect1d(g, top)) / K
        r = P2.replay_row(cur, g, K, head=0, stride=a.stride)
        f = int(np.count_nonzero(P2.keys(cur) >= np.uint32(r["Tc"])))
        recs.append((l, rho, j, alpha, r["I"], r["done"], f / K))
        print(f"layer {l:2d} rho {rho:.3f} draft {j} alpha {alpha:.3f}  I {r['I']:2d} done {r['done']} "
              f"f(Tc)/K {f / K:.3f} window [{r['L']},{r['H']}] count {r['count']}", flush=True)
    R = np.array([x[3:] for x in recs], dtype=np.float64)
    print(f"rows {len(recs)}: alpha mean {R[:, 0].mean():.3f}; I mean {R[:, 1].mean():.2f} max {R[:, 1].max():.0f}; "
          f"f/K mean {R[:, 3].mean():.3f} min {R[:, 3].min():.3f} max {R[:, 3].max():.3f}; "
          f"undershoot {(R[:, 3] < 1).sum()}; I hist {np.bincount(R[:, 1].astype(int)).tolist()}")


if __name__ == "__main__":
    main()
