#!/usr/bin/env python
"""Benchmark of the GVR exact Top-K hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl gvr|radix|reference]

A *step* is one pass of the whole hot path over one batch: one gvr_topk_batched launch
over all rows of the workload (BASELINE.json configs).  The default workload is
configs[1] (cfg2): 8 requests x 61 layers = 488 rows of N = 100,000 fp32 indexer
scores (Eq. 1, synthetic, prev-step guesses), K = 2048.  Inputs are resident
in HBM before the timed region; three distinct batches are rotated so every step reads
cold data (3 x 195 MB > 126 MB L2).  Rank 0 prints one JSON line.

A step of the default (batch filter) path launches four kernels of ours: gvr_guess_kernel
(Phases 1-2 for every row), gvr_filter_kernel (the one HBM pass, candidate lists),
gvr_refine_kernel (Phase 4 + ordered output per row) and gvr_fixup_kernel (rows the
lists cannot finish; usually none).  The roofline entry is for the dominant one (the
filter kernel), timed by CUDA events recorded on its stream through
gvr_topk_batched_events in a separate pass after the timed region (every 4th call);
roofline.whole_call is SURVEY 8(d)'s B(N) * R / elapsed over the whole call.

--gpus N > 1 without WORLD_SIZE re-runs this command under torch.distributed.run (one
rank per GPU, 127.0.0.1).  Under torchrun every rank processes its own batch of the same
shape (rows are independent; no collective on the hot path) — weak scaling; the elapsed
time is the max over ranks.  cfg5 instead splits one fixed 64 x 61 batch across the ranks
(paper_2604_22312_b200.shard.row_partition) — strong scaling.  --gather also times the
optional NCCL all-gather of out_idx, reported separately.  --impl reference times the
CPU oracle on the host (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K = 2048
CONFIGS = {
    "cfg1": dict(requests=1, layers=1, first_layer=30, n=8192, draft=1,
                 desc="single decode row N=8192 (layer 30, rho ~ 0.9)"),
    "cfg2": dict(requests=8, layers=61, n=100_000, draft=1, desc="batch 8 x 61 layers, N=100K"),
    "cfg3": dict(requests=1, layers=1, first_layer=30, n=131_072, draft=1,
                 desc="batch-1 long context N=131072 (layer 30, rho ~ 0.9); scripts/latency_sweep.py sweeps N"),
    "cfg4": dict(requests=16, layers=61, n=100_000, draft=4, desc="MTP-3: 16 requests x 4 tokens x 61 layers"),
    "cfg5": dict(requests=64, layers=61, n=131_072, draft=1, split=True,
                 desc="64 requests x 61 layers, N=128K, rows split across the GPUs"),
}
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


# ----------------------------------------------------------------------------- inputs
def make_decode_batch(requests, layers, n, dev, seed, draft=1, rank=0, first_layer=0, rho=None):
    """Synthetic decode batch: rows (request, layer, draft j) of length n + j from the
    Eq. 1 indexer (synth.IndexerLayer), plus prev_topk = the exact Top-K of the
    request's previous step (n - 1 keys), shared by its draft rows.
    Draft token j is one more AR(1) decode step of the query state than draft j - 1, so
    the shared guess gets staler along the draft.  rho overrides the
    per-layer AR coefficient (synth.layer_rho) for every layer.
    The previous step's Top-K is computed with the GVR kernel itself (no guess), i.e.
    the decode loop feeding its own output back; it is only a hint.
    `requests` is a count (requests 0..count-1) or an explicit list of global request
    ids (a rank's share of a split batch); `rank` enters the seed (weak scaling: every
    rank its own rows)."""
    import torch

    import paper_2604_22312_b200 as gvr
    import synth

    req_ids = list(range(requests)) if isinstance(requests, int) else list(requests)
    nreq = len(req_ids)
    R = nreq * layers * draft
    S = n + draft - 1
    scores = torch.zeros((R, S), dtype=torch.float32, device=dev)
    lens = torch.empty(R, dtype=torch.int32)
    prev_rows = torch.zeros((nreq * layers, S), dtype=torch.float32, device=dev)
    row = 0
    for qi, q in enumerate(req_ids):
        for li in range(layers):
            l = first_layer + li
            s = synth.splitmix64(seed, rank, q, l)
            lay = synth.IndexerLayer(S, synth.layer_rho(l, seed) if rho is None else rho, s, dev)
            prev_rows[qi * layers + li, :n - 1] = lay.scores(n - 1)
            lay.step()
            for j in range(draft):
                if j:
                    lay.step()
                scores[row, :n + j] = lay.scores(n + j)
                lens[row] = n + j
                row += 1
            del lay
    plens = torch.full((nreq * layers,), n - 1, dtype=torch.int32, device=dev)
    ptop = gvr.topk(prev_rows, K, row_lens=plens)
    prev = ptop.repeat_interleave(draft, dim=0).contiguous()
    del prev_rows
    return {"scores": scores, "row_lens": lens.to(dev), "prev": prev, "R": R, "n": n}


def algorithmic_bytes(lens, k=K):
    """Bytes the method must move per call: each row read once (4N), the guess read
    (4K), the output written (4K) and the row length (4) — SURVEY.md 8(d) B(N)."""
    return int(4 * int(np.sum(lens)) + len(lens) * (4 * k + 4 * k + 4))


def stream_kernel_bytes(lens, k=K, path="filter"):
    """Algorithmic bytes of the streaming kernel alone.  Filter path (gvr_filter_kernel):
    the row read once (4N) and the row length (4); its candidate lists are intermediate.
    Row path (gvr_topk_kernel): the row (4N), the output written (4K) and the row length.
    The guess read and its gathers belong to gvr_guess_kernel."""
    per_row = 4 if path == "filter" else 4 * k + 4
    return int(4 * int(np.sum(lens)) + len(lens) * per_row)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML in a background
    thread during the timed region (nvidia-smi's own sampler starts too slowly for a
    millisecond-scale region); falls back to nothing if NVML is unavailable."""

    def __init__(self, gpu_index, period_s: float = 0.002):
        self.gpu = int(gpu_index) if str(gpu_index).isdigit() else 0
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            time.sleep(0.01)
        except Exception:
            self._nvml = None
        return self

    def _run(self):
        p = self._nvml
        while not self._stop.is_set():
            try:
                sm = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
                rs = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def sample_now(self):
        if self._nvml is not None:
            p = self._nvml
            try:
                self.samples.append((p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM),
                                     p.nvmlDeviceGetCurrentClocksEventReasons(self._h)))
            except Exception:
                pass

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = set()
        for _, bits in self.samples:
            for b, name in REASON_BITS.items():
                if bits & b:
                    reasons.add(name)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml"}


# ----------------------------------------------------------------------------- timing
KERNEL_EVENT_EVERY = 4  # per-kernel events on every 4th timed step (each record costs ~2-3 us)


def time_steps(fn, batches, steps, warmup, stream, sampler=None, kernel_events=False, flush=None):
    """Device time of `steps` calls (seconds).  With kernel_events, every
    KERNEL_EVENT_EVERY-th call is fn(batch, evs), which also records per-kernel events on
    the launch stream; the mean per-kernel times (seconds per launch) are returned too.
    With `flush` (a device buffer larger than L2) every call is preceded by an untimed
    write of that buffer and timed alone with its own events (inputs smaller than L2)."""
    import torch
    for i in range(warmup):
        fn(batches[i % len(batches)])
    torch.cuda.synchronize()
    if flush is not None:
        total, kern, nk = 0.0, {"guess": 0.0, "stream": 0.0, "refine": 0.0}, 0
        for i in range(steps):
            flush.fill_(float(i))  # write-only flush (the contract's "write a buffer larger than L2")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            kev = ([torch.cuda.Event(enable_timing=True) for _ in range(4)]
                   if kernel_events and i % KERNEL_EVENT_EVERY == 0 else None)
            e0.record(stream)
            if kev is not None:
                fn(batches[i % len(batches)], kev)
            else:
                fn(batches[i % len(batches)])
            e1.record(stream)
            if sampler is not None and i == steps // 2:
                sampler.sample_now()
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1) / 1e3
            if kev is not None:
                kern["guess"] += kev[0].elapsed_time(kev[1]) / 1e3
                kern["stream"] += kev[1].elapsed_time(kev[2]) / 1e3
                kern["refine"] += kev[2].elapsed_time(kev[3]) / 1e3
                nk += 1
        if not kernel_events:
            return total
        return total, {k: v / max(nk, 1) for k, v in kern.items()} | {"sampled_steps": nk}
    sampled = [i for i in range(steps) if i % KERNEL_EVENT_EVERY == 0] if kernel_events else []
    evs = {i: [torch.cuda.Event(enable_timing=True) for _ in range(4)] for i in sampled}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(steps):
        if i in evs:
            fn(batches[i % len(batches)], evs[i])
        else:
            fn(batches[i % len(batches)])
    ev1.record(stream)
    if sampler is not None:
        sampler.sample_now()  # GPU still executing the queued steps
    torch.cuda.synchronize()
    total = ev0.elapsed_time(ev1) / 1e3
    if not kernel_events:
        return total
    def mean(a, b):
        return sum(e[a].elapsed_time(e[b]) for e in evs.values()) / 1e3 / len(evs)
    return total, {"guess": mean(0, 1), "stream": mean(1, 2), "refine": mean(2, 3), "sampled_steps": len(evs)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_rate(host_scores, lens, max_rows=None, threads=None):
    import oracle
    rows = host_scores if max_rows is None else host_scores[:max_rows]
    ln = lens if max_rows is None else lens[:max_rows]
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.topk_batched(rows, K, row_lens=ln, num_threads=threads)
    dt = time.perf_counter() - t0
    return rows.shape[0] / dt, threads, rows.shape[0], dt


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="gvr", choices=["gvr", "radix", "radix2", "reference"])
    ap.add_argument("--nbatches", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", action="store_true", help="verify every batch against the oracle")
    ap.add_argument("--path", default="filter", choices=["filter", "row"],
                    help="batch path of the library (gvr_options.batch_path): filter kernel + refine, or row kernel")
    ap.add_argument("--gather", action="store_true",
                    help="N > 1: also time the optional NCCL all-gather of out_idx (reported separately)")
    ap.add_argument("--cpu-dry-run", action="store_true",
                    help="launcher / rank-plumbing check without a GPU: gloo process group, no kernels")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this command under torch.distributed.run (rank 0 prints)
        return launch_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if args.cpu_dry_run:
        return run_dry(args, cfg, rank, world)

    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2604_22312_b200 as gvr
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    split = bool(cfg.get("split"))
    if split:
        # strong scaling: the global batch is fixed, each rank owns a contiguous block of
        # requests (equal rows, so the row_partition is by request)
        from paper_2604_22312_b200.shard import row_partition
        qb = row_partition(np.full(cfg["requests"], cfg["n"]), world)
        reqs, seed_rank = list(range(int(qb[rank]), int(qb[rank + 1]))), 0
    else:
        reqs, seed_rank = cfg["requests"], rank
    batches = [make_decode_batch(reqs, cfg["layers"], cfg["n"], dev,
                                 seed=synth.splitmix64(synth.BASE_SEED, b), draft=cfg["draft"], rank=seed_rank,
                                 first_layer=cfg.get("first_layer", 0))
               for b in range(args.nbatches)]
    torch.cuda.synchronize()
    R = batches[0]["R"]
    lens_np = batches[0]["row_lens"].cpu().numpy()
    stream = torch.cuda.current_stream()
    for b in batches:
        b["out"] = torch.empty((R, K), dtype=torch.int32, device=dev)

    opts = None
    if args.path == "row":
        opts = gvr.GvrOptions(float("nan"), 0, 0, 0, 1)

    def gvr_step(b, evs=None):
        if evs is None:
            gvr.topk(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], out=b["out"], options=opts)
        else:
            gvr.topk_events(b["scores"], K, row_lens=b["row_lens"], prev=b["prev"], out=b["out"], events=evs,
                            options=opts)

    def radix_step(b):
        gvr.radix_topk(b["scores"], K, row_lens=b["row_lens"], out=b["out"])

    def radix2_step(b):
        gvr.radix2_topk(b["scores"], K, row_lens=b["row_lens"], out=b["out"])

    main_fn = {"gvr": gvr_step, "radix": radix_step, "radix2": radix2_step}[args.impl]
    other_fn = radix_step if args.impl == "gvr" else gvr_step

    # correctness gate (oracle) on one batch before timing
    check = {}
    if rank == 0:
        import oracle
        b0 = batches[0]
        main_fn(b0)
        torch.cuda.synchronize()
        host0 = b0["scores"].cpu().numpy()
        ref = oracle.topk_batched(host0, K, row_lens=lens_np)
        ok = bool(np.array_equal(b0["out"].cpu().numpy(), ref))
        check = {"bit_exact_vs_oracle": ok, "rows_checked": int(R)}
        if not ok:
            print(json.dumps({"error": "parity failure vs oracle", "config": args.config}), flush=True)
            sys.exit(2)

    # timed region
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = vis.split(",")[local_rank] if vis else str(local_rank)
    kern_times = None
    batch_bytes = sum(int(b["scores"].numel()) * 4 for b in batches)
    flush = None
    if batch_bytes < 2 * 126 * 2**20:  # rotated inputs fit in L2: flush before every call
        flush = torch.zeros(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    info = gvr.kernel_info()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fused = R <= info["gvr"]["ctas_per_sm"] * sms  # one wave: the library's single-kernel path
    with ClockSampler(phys) as clk:
        if args.impl == "gvr" and fused:
            # the call is one kernel (gvr_topk_kernel, Phase 1 inside): its call events time it
            elapsed = time_steps(main_fn, batches, args.steps, args.warmup, stream, sampler=clk, flush=flush)
            kern_times = {"guess": 0.0, "stream": elapsed / args.steps, "refine": 0.0,
                          "sampled_steps": args.steps}
        elif args.impl == "gvr":
            # the timed region runs the calls as a user would (programmatic dependent launch
            # between the kernels); per-kernel times come from a separate pass whose calls
            # record events between the kernels (which serialises them)
            elapsed = time_steps(main_fn, batches, args.steps, args.warmup, stream, sampler=clk, flush=flush)
            _, kern_times = time_steps(main_fn, batches, args.steps, 0, stream, kernel_events=True, flush=flush)
        else:
            elapsed = time_steps(main_fn, batches, args.steps, args.warmup, stream, sampler=clk, flush=flush)
    if dist is not None:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    ms_per_step = elapsed / args.steps * 1e3
    rows_all = R
    if dist is not None:
        t = torch.tensor([R], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        rows_all = int(t.item())
    rows_total = rows_all * args.steps
    value = rows_total / elapsed

    # the other kernel, same protocol (speedup vs own radix select), and the same-geometry
    # radix baseline (radix2: histogram pass + the GVR filter / refine machinery)
    other_elapsed = time_steps(other_fn, batches, args.steps, args.warmup, stream, flush=flush)
    r2_elapsed = (time_steps(radix2_step, batches, args.steps, args.warmup, stream, flush=flush)
                  if args.impl == "gvr" else None)
    if dist is not None:
        t = torch.tensor([other_elapsed, r2_elapsed or 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        other_elapsed = float(t[0].item())
        r2_elapsed = float(t[1].item()) if r2_elapsed is not None else None

    # optional all-gather of every rank's indices (off the hot path, timed separately)
    gather_info = None
    if dist is not None and args.gather:
        from paper_2604_22312_b200.shard import gather_rows
        sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([R], dtype=torch.int64, device=dev))
        bounds = np.concatenate([[0], np.cumsum([int(x.item()) for x in sizes])])
        for _ in range(3):
            gather_rows(batches[0]["out"], bounds)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(10):
            full = gather_rows(batches[0]["out"], bounds)
        g1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([g0.elapsed_time(g1) / 10 * 1e3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather_info = {"allgather_us": round(float(t.item()), 2), "bytes_out": int(full.numel() * 4),
                       "collective": "torch.distributed.all_gather (NCCL)"}

    # per-row stats (passes etc.) on one batch, outside the timed region
    b0 = batches[0]
    if args.impl == "gvr":
        _, _, st = gvr.topk_ex(b0["scores"], K, row_lens=b0["row_lens"], prev=b0["prev"], values=False)
    elif args.impl == "radix2":
        _, _, st = gvr.radix2_topk_ex(b0["scores"], K, row_lens=b0["row_lens"], values=False)
    else:
        _, _, st = gvr.radix_topk_ex(b0["scores"], K, row_lens=b0["row_lens"], values=False)
    st = st.cpu().numpy()

    result = None
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
        abytes = algorithmic_bytes(lens_np)
        G = int(st[:, 7].max()) if args.impl == "gvr" else 1  # CTAs per row (stats.cluster)
        if fused and G > 1:
            stream_kernel, n_kernels = "gvr_topk_cluster_kernel", 1
            gvr_path = f"cluster kernel: {G} CTAs per row merged through DSMEM (few long rows)"
        elif fused:
            stream_kernel, n_kernels, gvr_path = "gvr_topk_kernel", 1, "fused single kernel (one wave)"
        elif args.path == "filter":
            stream_kernel, n_kernels = "gvr_filter_kernel", 4  # guess, filter, refine, fixup
            gvr_path = ("guess kernel + filter kernel (whole batch, one HBM pass) + refine kernel (rows from their "
                        "candidate lists) + fixup kernel (rows the lists cannot finish; usually none)")
        else:
            stream_kernel, n_kernels, gvr_path = "gvr_topk_kernel", 2, "guess kernel + row streaming kernel"

        def kernel_us(kt):
            names = {"guess": "gvr_guess_kernel", "stream": stream_kernel,
                     "refine": "gvr_refine_kernel + gvr_fixup_kernel" if stream_kernel == "gvr_filter_kernel"
                     else None}
            d = {names[k]: round(kt[k] * 1e6, 2) for k in ("guess", "stream", "refine") if names[k]}
            return d | {"sampled_steps": kt["sampled_steps"]}
        step_gbs = abytes / (elapsed / args.steps) / 1e9  # whole call (all kernels + gaps)
        if args.impl == "gvr":
            # dominant kernel: the streaming / refine kernel, timed by its own events
            kbytes = stream_kernel_bytes(lens_np, path=args.path) if not fused else abytes
            kern_s = kern_times["stream"]
        else:
            kbytes = abytes  # the radix kernel is the whole call
            kern_s = elapsed / args.steps
        achieved = kbytes / kern_s / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                traffic = json.load(open(tf)).get(f"{args.impl}_{args.config}")
            except Exception:
                traffic = None
        gvr_t = elapsed if args.impl == "gvr" else other_elapsed
        rad_t = other_elapsed if args.impl == "gvr" else elapsed
        result = {
            "metric": "µs/row & rows/s, K=2048 N=100K; speedup vs own radix-select; HBM GB/s",
            "value": round(value, 1),
            "unit": "rows/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "strong" if split else "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (PAPER.md Eq. 1 indexer rows, YaRN RoPE, AR(1) decode steps; prev-step Top-K guesses)",
            "impl": args.impl,
            "config": {"workload": f"{args.config}: {cfg['desc']}", "rows_per_gpu": R, "N": cfg["n"], "K": K,
                       "draft_tokens": cfg["draft"], "parallelism": f"row-shard x{world}",
                       "l2": (f"inputs larger than L2: {args.nbatches} distinct batches rotated "
                              f"({batch_bytes / 1e6:.0f} MB)") if flush is None else
                             (f"inputs ({batch_bytes / 1e6:.2f} MB) fit in L2: a 256 MB buffer is written before "
                              f"every call (untimed), each call timed alone with CUDA events")},
            "us_per_row": round(elapsed / (R * args.steps) * 1e6, 5),
            "speedup_vs_radix": round(rad_t / gvr_t, 3),
            "radix_rows_per_s": round(rows_all * args.steps / rad_t, 1),
            # the same-geometry radix (radix2_topk_batched: one half-digit histogram pass +
            # the GVR filter / refine machinery): the fair comparison
            "speedup_vs_radix_same_geometry": (round(r2_elapsed / gvr_t, 3) if r2_elapsed else None),
            "radix2_rows_per_s": (round(rows_all * args.steps / r2_elapsed, 1) if r2_elapsed else None),
            "radix_baselines": {"radix": "radix_topk_batched: one CTA per row, 11/11/10-bit rounds re-reading "
                                         "the row, early exit (PAPER.md:125-148)",
                                "radix2": "radix2_topk_batched: persistent TMA stream of the half digit "
                                          "histogram, then the GVR filter at the K-th bin and the GVR refine"},
            "hbm_gbs": round(step_gbs, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": kbytes,
                         "kernel": stream_kernel if args.impl == "gvr" else f"{args.impl}_topk (whole call)",
                         "kernel_us_per_launch": round(kern_s * 1e6, 2),
                         "step_gbs": round(step_gbs, 1),
                         # SURVEY 8(d)'s definition over the whole call: B(N) * R / elapsed
                         "whole_call": {"achieved": round(step_gbs, 1), "frac": round(step_gbs / peak, 4),
                                        "algorithmic_bytes_per_call": abytes}},
            "kernel_us_per_launch": (kernel_us(kern_times) if kern_times else None),
            "passes_per_row": {"global_mean": float(st[:, 4].mean()), "secant_mean": float(st[:, 0].mean()),
                               "snap_mean": float(st[:, 1].mean()), "raises_mean": float(st[:, 5].mean()),
                               "cand_mean": float(st[:, 2].mean())},
            "gpu_launches": args.steps * (n_kernels if args.impl == "gvr" else (5 if args.impl == "radix2" else 1)),
            "gvr_path": gvr_path if args.impl == "gvr" else None,
            "clocks": clk.summary(),
            "allgather": gather_info,
            "check": check,
        }
    # end-to-end through the host-buffer C ABI (H2D + kernel + D2H in the timed region)
    if rank == 0 and not args.no_e2e and args.impl == "gvr":
        result["e2e"] = run_e2e(gvr, batches[0], args, dev)
    if rank == 0 and not args.no_cpu:
        host0 = batches[0]["scores"].cpu().numpy()
        rate, threads, nrows, dt = cpu_oracle_rate(host0, lens_np)
        n1 = min(8, nrows)
        rate1, _, _, dt1 = cpu_oracle_rate(host0, lens_np, max_rows=n1, threads=1)
        result["cpu_baseline"] = {"value": round(rate, 2), "unit": "rows/s", "cores": threads, "kind": "oracle",
                                  "sample": f"{nrows} rows of {args.config} (one full batch), qsort oracle, "
                                            f"{dt:.2f} s wall on {threads} threads",
                                  "single_thread_ms_per_row": round(dt1 / n1 * 1e3, 3),
                                  "cpu_model": cpu_model()}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def launch_ranks(n):
    """`bench.py --gpus N` without WORLD_SIZE: start N ranks on this node with
    torch.distributed.run (rendezvous on 127.0.0.1, a free port) and wait for them."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)


def run_dry(args, cfg, rank, world):
    """--cpu-dry-run: the multi-rank plumbing of the real run (process group, barrier +
    max-over-ranks timing, aggregate rows/s, rank-0 JSON line) on gloo without kernels; the
    per-rank work is the config's row partition with a host-side stand-in step."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    split = bool(cfg.get("split"))
    from paper_2604_22312_b200.shard import row_partition
    per_req = cfg["layers"] * cfg["draft"]
    if split:  # strong scaling: contiguous blocks of requests, as in the real run
        qb = row_partition(np.full(cfg["requests"], cfg["n"]), world)
        R = int(qb[rank + 1] - qb[rank]) * per_req
    else:
        R = cfg["requests"] * per_req
    x = np.random.default_rng(rank).standard_normal((min(R, 8), 4096)).astype(np.float32)
    for _ in range(args.warmup):
        np.sort(x, axis=1)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        np.sort(x, axis=1)
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
        n = torch.tensor([R], dtype=torch.int64)
        dist.all_reduce(n)
        rows_all = int(n.item())
    else:
        rows_all = R
    if rank == 0:
        print(json.dumps({"metric": "dry run (no kernels)", "value": round(rows_all * args.steps / el, 1),
                          "unit": "rows/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "scaling": "strong" if split else "weak", "rows_per_rank0": R, "rows_all": rows_all,
                          "config": {"workload": args.config}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(gvr, batch, args, dev):
    import torch
    R = batch["R"]
    S = batch["scores"].shape[1]
    h_scores = torch.empty((R, S), dtype=torch.float32, pin_memory=True)
    h_scores.copy_(batch["scores"].cpu())
    h_prev = torch.empty((R, K), dtype=torch.int32, pin_memory=True)
    h_prev.copy_(batch["prev"].cpu())
    h_lens = torch.empty(R, dtype=torch.int32, pin_memory=True)
    h_lens.copy_(batch["row_lens"].cpu())
    h_out = torch.empty((R, K), dtype=torch.int32, pin_memory=True)
    ws = gvr.Workspace(R, S, K)
    stream = torch.cuda.current_stream()
    steps = max(3, min(args.steps, 10))

    def step():
        gvr.topk_host_ptr(h_scores.data_ptr(), S, R, ws, K, h_out.data_ptr(), prev_ptr=h_prev.data_ptr(),
                          lens_ptr=h_lens.data_ptr(), stream=stream)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / 1e3
    ws.close()
    return {"value": round(R * steps / dt, 1), "unit": "rows/s",
            "h2d_bytes_per_step": int(R * S * 4 + R * K * 4 + R * 4),
            "d2h_bytes_per_step": int(R * K * 4), "steps": steps,
            "api": "gvr_topk_batched_host (C ABI, pinned host buffers)"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores, rank 0 only.
    Each step is a bounded sample of the workload (SAMPLE rows of the config)."""
    if rank != 0:
        return
    import torch

    import synth
    torch.set_num_threads(os.cpu_count() or 1)
    sample_rows = 16
    n = cfg["n"]
    rows, lens = [], []
    r = 0
    for l in range(cfg["layers"]):
        if r >= sample_rows:
            break
        lay = synth.IndexerLayer(n + cfg["draft"] - 1, synth.layer_rho(l, synth.BASE_SEED),
                                 synth.splitmix64(synth.BASE_SEED, 0, 0, l), "cpu")
        lay.step()
        for j in range(cfg["draft"]):
            if r >= sample_rows:
                break
            row = np.zeros(n + cfg["draft"] - 1, np.float32)
            row[:n + j] = lay.scores(n + j).numpy()
            rows.append(row)
            lens.append(n + j)
            r += 1
    host = np.stack(rows)
    lens = np.array(lens, np.int32)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_rate(host, lens, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_oracle_rate(host, lens, threads=threads)
    dt = time.perf_counter() - t0
    value = host.shape[0] * args.steps / dt
    sample = f"{host.shape[0]} rows of {args.config} per step (N={n}), qsort oracle on {threads} threads"
    print(json.dumps({
        "metric": "µs/row & rows/s, K=2048 N=100K; speedup vs own radix-select; HBM GB/s",
        "value": round(value, 2), "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "N": n, "K": K},
        "cpu_baseline": {"value": round(value, 2), "unit": "rows/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 2), "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
