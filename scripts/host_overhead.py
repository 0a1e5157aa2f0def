"""Host (CPU) time per call of each entry path, measured without synchronising: if it
exceeds the GPU time per call the GPU starves and the loop is launch-bound."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2604_22312_b200 as gvr
dev = torch.device("cuda:0")
b = bench.make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED)
out = torch.empty((b["R"], bench.K), dtype=torch.int32, device=dev)
lib = gvr.library()
S = b["scores"].shape[1]
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (ctypes.c_void_p(b["scores"].data_ptr()), S, ctypes.c_void_p(b["row_lens"].data_ptr()), b["R"],
        ctypes.c_void_p(b["prev"].data_ptr()), bench.K, ctypes.c_void_p(out.data_ptr()), sp)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
paths = {
    "ctypes direct": lambda: lib.gvr_topk_batched(*args),
    "gvr.topk": lambda: gvr.topk(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out),
    "gvr.topk_events": lambda: gvr.topk_events(b["scores"], bench.K, row_lens=b["row_lens"], prev=b["prev"], out=out, events=evs),
    "empty torch op": lambda: out.zero_(),
}
for name, fn in paths.items():
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:18s} host {1e6*(t1-t0)/n:8.1f} us/call   wall incl. drain {1e6*(t2-t0)/n:8.1f} us/call", flush=True)
