"""cfg2 (or another bench config) time per step with force_cluster = 1, 2, 4, 8."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2604_22312_b200 as gvr
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--gs", default="0,1,2,4")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda:0")
bs = [bench.make_decode_batch(cfg["requests"], cfg["layers"], cfg["n"], dev, seed=synth.splitmix64(synth.BASE_SEED, i),
                              draft=cfg["draft"]) for i in range(3)]
out = torch.empty((bs[0]["R"], bench.K), dtype=torch.int32, device=dev)
for G in [int(x) for x in args.gs.split(",")]:
    opt = gvr.GvrOptions(float("nan"), 0, G, 0)
    def step(i):
        b = bs[i % 3]
        gvr.topk_ex(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out, values=False, stats=False,
                    options=opt)
    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(30):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    print(f"force_cluster={G}: {e0.elapsed_time(e1) / 30 * 1e3:.1f} us/step", flush=True)
