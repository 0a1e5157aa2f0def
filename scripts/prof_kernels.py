"""Profiling driver: build one cfg2 batch, run GVR and radix a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import bench, synth
import paper_2604_22312_b200 as gvr

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
b = bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.BASE_SEED, draft=cfg["draft"])
torch.cuda.synchronize()
out = torch.empty((b["R"], bench.K), dtype=torch.int32, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for i in range(args.iters):
    flush.zero_()
    gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out)
    flush.zero_()
    gvr.radix_topk(b["scores"], bench.K, row_lens=b["row_lens"], out=out)
torch.cuda.synchronize()
print("done")
