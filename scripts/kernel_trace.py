"""Device-side timeline of a few GVR steps via torch.profiler (CUPTI): every kernel /
memcpy / memset with its start offset and duration, to find gaps between launches."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2604_22312_b200 as gvr
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--impl", default="gvr")
ap.add_argument("--case", default=None, help="worst_cases.py batch kind:guess, e.g. ties90:random")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
if args.case:
    import numpy as np
    kind, gk = args.case.split(":")
    R, N = 488, 100_000
    def dist_batch(seed):
        s = torch.from_numpy(np.stack([synth.dist_row(kind, N, seed=seed + r) for r in range(R)])).to(dev)
        if gk == "adversarial":
            prev = torch.argsort(s, dim=1, stable=True)[:, :bench.K].to(torch.int32).contiguous()
        else:
            prev = torch.randint(0, N, (R, bench.K), dtype=torch.int32, device=dev,
                                 generator=torch.Generator(dev).manual_seed(seed))
        return {"scores": s, "row_lens": torch.full((R,), N, dtype=torch.int32, device=dev), "prev": prev, "R": R}
    bs = [dist_batch(9000 + 1000 * i) for i in range(3)]
    _, _, st = gvr.topk_ex(bs[0]["scores"], bench.K, row_lens=bs[0]["row_lens"], prev=bs[0]["prev"])
    st = st.cpu().numpy()
    for i, f in enumerate(gvr.STATS_FIELDS):
        print(f"{f:14s} mean {st[:, i].mean():10.2f} min {st[:, i].min():10d} max {st[:, i].max():10d}")
else:
    bs = [bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.splitmix64(synth.BASE_SEED, i),
                                  draft=cfg["draft"]) for i in range(3)]
out = torch.empty((bs[0]["R"], bench.K), dtype=torch.int32, device=dev)
it = [0]
def step():
    b = bs[it[0] % 3]
    it[0] += 1
    if args.impl == "gvr":
        gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out)
    else:
        gvr.radix_topk(b["scores"], bench.K, row_lens=b["row_lens"], out=out)
for _ in range(5):
    step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(6):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
prev_end = None
for e in evs:
    st, du = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = "" if prev_end is None else f" gap {st - prev_end:7.1f}"
    print(f"{st:9.1f} us  dur {du:8.1f}{gap}  {e.name[:70]}")
    prev_end = st + du
