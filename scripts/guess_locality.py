"""How many distinct 32-B / 64-B DRAM segments do a row's 2048 guessed positions touch?
(If top-K positions cluster, index-sorted gathers would share sectors.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
prev = b["prev"].cpu().numpy()
s32, s64 = [], []
for r in range(0, b["R"], 7):
    p = prev[r][prev[r] >= 0]
    s32.append(len(np.unique(p // 8)) / len(p))
    s64.append(len(np.unique(p // 16)) / len(p))
print(f"distinct 32B sectors per gather: mean {np.mean(s32):.3f} min {np.min(s32):.3f}; 64B segments: mean {np.mean(s64):.3f} min {np.min(s64):.3f}")
