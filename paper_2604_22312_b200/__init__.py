"""paper_2604_22312_b200 — B200-native GVR exact Top-K (arXiv 2604.22312).

Thin ctypes binding over the C ABI of ``libgvrtopk.so`` (declared in
``include/gvr_topk.h``).  This module only marshals arguments: every step of the
Top-K path runs in the CUDA kernels of the shared library.  There is no CPU or
PyTorch fallback — if the library or a CUDA device is missing, calls raise.

    topk(scores, k=2048, row_lens=None, prev=None)   -> int32 [R, k] (GVR)
    radix_topk(scores, k=2048, row_lens=None)         -> int32 [R, k] (radix baseline)
    radix2_topk(scores, k=2048, row_lens=None)        -> int32 [R, k] (same-geometry radix)
    topk_ex(...)                                      -> (idx, values, stats)
    topk_host(scores_np, ...)                         -> host-buffer C-ABI entry point

``scores`` is a CUDA fp32 tensor [R, S] whose last dim is contiguous (any row
stride); ``row_lens`` an int32 CUDA tensor [R] or None; ``prev`` an int32 CUDA tensor
[R, k] (the previous decode step's Top-K) or None.  Output order: score descending,
index ascending; rows shorter than k are padded with -1.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgvrtopk.so")
_lib = None

STATS_FIELDS = ("secant_iters", "snap_iters", "cand_count", "done_kind", "global_passes",
                "raises", "buffer_count", "cluster", "phase2_exit", "sample_count", "tc_key", "reserved")
PHASE2_EXITS = {0: "all", 1: "window", 2: "ties", 3: "exhausted"}
DONE_KINDS = {0: "trivial", 1: "converged", 2: "tiefill", 3: "radix"}
MAX_K = 2048


class GvrOptions(ctypes.Structure):
    _fields_ = [("window_z", ctypes.c_float), ("max_secant_iters", ctypes.c_int32),
                ("force_cluster", ctypes.c_int32), ("guess_stride", ctypes.c_int32),
                ("batch_path", ctypes.c_int32)]


class GvrError(RuntimeError):
    pass


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GvrError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    sigs = {
        "gvr_topk_batched": [vp, i64, vp, i32, vp, i32, vp, vp],
        "gvr_topk_batched_ex": [vp, i64, vp, i32, vp, i32, vp, vp, vp, vp, vp],
        "radix_topk_batched": [vp, i64, vp, i32, i32, vp, vp],
        "radix_topk_batched_ex": [vp, i64, vp, i32, i32, vp, vp, vp, vp],
        "radix2_topk_batched": [vp, i64, vp, i32, i32, vp, vp],
        "gvr_indexer_scores": [vp, i64, vp, vp, vp, vp, i32, vp, i64, vp],
        "gvr_indexer_topk_batched": [vp, i64, vp, vp, vp, vp, i32, vp, i32, vp, vp, vp],
        "radix2_topk_batched_ex": [vp, i64, vp, i32, i32, vp, vp, vp, vp],
        "gvr_workspace_create": [i32, i64, i32, ctypes.POINTER(vp)],
        "gvr_workspace_destroy": [vp],
        "gvr_topk_batched_host": [vp, i64, vp, i32, vp, i32, vp, vp, vp],
        "gvr_topk_phase_timing": [vp, i64, vp, i32, vp, i32, vp, vp, vp],
        "gvr_topk_batched_events": [vp, i64, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.gvr_status_string.argtypes = [ctypes.c_int]
    lib.gvr_status_string.restype = ctypes.c_char_p
    lib.gvr_last_cuda_error.argtypes = []
    lib.gvr_last_cuda_error.restype = ctypes.c_char_p
    lib.gvr_version.argtypes = []
    lib.gvr_version.restype = ctypes.c_int32
    lib.gvr_cta_timeline.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                     ctypes.POINTER(ctypes.c_int32)]
    lib.gvr_cta_timeline.restype = ctypes.c_int
    lib.gvr_kernel_info.argtypes = [ctypes.POINTER(ctypes.c_int32)] * 6
    lib.gvr_kernel_info.restype = ctypes.c_int
    _lib = lib
    return lib


def library():
    """The loaded ctypes library (loads it on first use)."""
    return _load()


def cta_timeline(enable: bool, kernel: str = "filter", max_ctas: int = 4096):
    """gvr_cta_timeline: enable=True starts recording the filter path's CTA timeline;
    enable=False stops and returns an int64 array [n, 4] for kernel "filter" (entry ns,
    after the Phase-1/2 wait ns, exit ns, SM id) or "guess" (entry ns, exit ns, loads arrived ns, Phase 1 done ns).
    Call enable=False once per kernel wanted (the first call stops recording)."""
    import numpy as np
    kid = {"filter": 0, "guess": 1}[kernel]
    if enable:
        _check(_load().gvr_cta_timeline(kid, 1, None, 0, None))
        return None
    out = np.zeros((max_ctas, 4), dtype=np.int64)
    n = ctypes.c_int32(0)
    _check(_load().gvr_cta_timeline(kid, 0, out.ctypes.data, max_ctas, ctypes.byref(n)))
    return out[:n.value]


def kernel_info() -> dict:
    """Resident CTAs per SM, threads and dynamic shared memory of both kernels (current device)."""
    v = [ctypes.c_int32(0) for _ in range(6)]
    _check(_load().gvr_kernel_info(*[ctypes.byref(x) for x in v]))
    return {"gvr": {"ctas_per_sm": v[0].value, "threads": v[1].value, "smem_bytes": v[2].value},
            "radix": {"ctas_per_sm": v[3].value, "threads": v[4].value, "smem_bytes": v[5].value}}


def _check(rc: int):
    if rc != 0:
        msg = _load().gvr_status_string(rc).decode()
        if rc == 3:
            msg += ": " + _load().gvr_last_cuda_error().decode()
        raise GvrError(msg)


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _prep(scores, k, row_lens, prev, out):
    torch = _torch()
    if not isinstance(scores, torch.Tensor) or not scores.is_cuda:
        raise GvrError("scores must be a CUDA tensor (no CPU path)")
    if scores.dtype != torch.float32 or scores.dim() != 2 or scores.stride(1) != 1:
        raise GvrError("scores must be fp32 [R, S] with a contiguous last dim")
    R = scores.shape[0]
    stride = scores.stride(0) if R > 1 else max(scores.shape[1], 1)
    if row_lens is not None:
        if row_lens.dtype != torch.int32 or row_lens.shape != (R,) or not row_lens.is_cuda:
            raise GvrError("row_lens must be int32 CUDA [R]")
        row_lens = row_lens.contiguous()
    elif scores.shape[1] != stride:
        row_lens = torch.full((R,), scores.shape[1], dtype=torch.int32, device=scores.device)
    if prev is not None:
        if prev.dtype != torch.int32 or prev.shape != (R, k) or not prev.is_cuda or not prev.is_contiguous():
            raise GvrError("prev must be a contiguous int32 CUDA tensor [R, k]")
    if out is None:
        out = torch.empty((R, k), dtype=torch.int32, device=scores.device)
    elif out.dtype != torch.int32 or out.shape != (R, k) or not out.is_contiguous():
        raise GvrError("out must be a contiguous int32 tensor [R, k]")
    return R, stride, row_lens, prev, out


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def topk(scores, k: int = MAX_K, row_lens=None, prev=None, out=None, stream=None, options=None):
    """GVR exact ordered Top-K of every row (launch is stream-ordered, no host sync)."""
    R, stride, row_lens, prev, out = _prep(scores, k, row_lens, prev, out)
    if options is None:
        _check(_load().gvr_topk_batched(_ptr(scores), stride, _ptr(row_lens), R, _ptr(prev), k,
                                        _ptr(out), _stream_ptr(stream)))
    else:
        _check(_load().gvr_topk_batched_ex(_ptr(scores), stride, _ptr(row_lens), R, _ptr(prev), k,
                                           _ptr(out), _stream_ptr(stream), ctypes.byref(options), None, None))
    return out


def topk_ex(scores, k: int = MAX_K, row_lens=None, prev=None, out=None, values: bool = True,
            stats: bool = True, options: GvrOptions | None = None, stream=None):
    """GVR Top-K plus optional selected values [R, k] and per-row stats [R, 12] (int32,
    columns STATS_FIELDS; tc_key is the uint32 bit pattern)."""
    torch = _torch()
    R, stride, row_lens, prev, out = _prep(scores, k, row_lens, prev, out)
    val = torch.empty((R, k), dtype=torch.float32, device=scores.device) if values else None
    st = torch.zeros((R, len(STATS_FIELDS)), dtype=torch.int32, device=scores.device) if stats else None
    opt = ctypes.byref(options) if options is not None else None
    _check(_load().gvr_topk_batched_ex(_ptr(scores), stride, _ptr(row_lens), R, _ptr(prev), k,
                                       _ptr(out), _stream_ptr(stream), opt, _ptr(val), _ptr(st)))
    return out, val, st


PHASES = ("phase1", "stream", "phase2_3", "phase4", "output")


def topk_events(scores, k: int = MAX_K, row_lens=None, prev=None, out=None, events=(None, None, None, None),
                stream=None, options=None):
    """gvr.topk that also records four torch.cuda.Events (each may be None): before the
    guess kernel, before and after the streaming kernel (gvr_filter_kernel on the batch
    filter path, else gvr_topk_kernel) and at the end of the call."""
    R, stride, row_lens, prev, out = _prep(scores, k, row_lens, prev, out)
    hs = []
    events = tuple(events) + (None,) * (4 - len(events))
    for e in events:
        if e is None:
            hs.append(None)
        else:
            if e.cuda_event == 0:  # created lazily by torch: force creation
                e.record()
            hs.append(ctypes.c_void_p(e.cuda_event))
    opt = ctypes.byref(options) if options is not None else None
    _check(_load().gvr_topk_batched_events(_ptr(scores), stride, _ptr(row_lens), R, _ptr(prev), k, _ptr(out),
                                           _stream_ptr(stream), *hs, opt))
    return out


def topk_phase_timing(scores, k: int = MAX_K, row_lens=None, prev=None, out=None, stream=None):
    """GVR Top-K plus per-row stamps [R, 9]: clock64 at start, end of Phase 1, stream,
    Phases 2-3, Phase 4, end — the paper's per-phase breakdown (Table 8) — then the
    global timer (ns) at the CTA's start and end and the SM id."""
    torch = _torch()
    R, stride, row_lens, prev, out = _prep(scores, k, row_lens, prev, out)
    ts = torch.zeros((R, 9), dtype=torch.int64, device=scores.device)
    _check(_load().gvr_topk_phase_timing(_ptr(scores), stride, _ptr(row_lens), R, _ptr(prev), k,
                                         _ptr(out), _stream_ptr(stream), _ptr(ts)))
    return out, ts


def radix_topk(scores, k: int = MAX_K, row_lens=None, out=None, stream=None):
    """Radix-select baseline with the same output contract."""
    R, stride, row_lens, _, out = _prep(scores, k, row_lens, None, out)
    _check(_load().radix_topk_batched(_ptr(scores), stride, _ptr(row_lens), R, k, _ptr(out),
                                      _stream_ptr(stream)))
    return out


def radix_topk_ex(scores, k: int = MAX_K, row_lens=None, out=None, values=True, stats=True, stream=None):
    torch = _torch()
    R, stride, row_lens, _, out = _prep(scores, k, row_lens, None, out)
    val = torch.empty((R, k), dtype=torch.float32, device=scores.device) if values else None
    st = torch.zeros((R, len(STATS_FIELDS)), dtype=torch.int32, device=scores.device) if stats else None
    _check(_load().radix_topk_batched_ex(_ptr(scores), stride, _ptr(row_lens), R, k, _ptr(out),
                                         _stream_ptr(stream), _ptr(val), _ptr(st)))
    return out, val, st


def radix2_topk(scores, k: int = MAX_K, row_lens=None, out=None, stream=None):
    """Same-geometry radix baseline (histogram pass + GVR filter / refine machinery)."""
    R, stride, row_lens, _, out = _prep(scores, k, row_lens, None, out)
    _check(_load().radix2_topk_batched(_ptr(scores), stride, _ptr(row_lens), R, k, _ptr(out), _stream_ptr(stream)))
    return out


def radix2_topk_ex(scores, k: int = MAX_K, row_lens=None, out=None, values=True, stats=True, stream=None):
    torch = _torch()
    R, stride, row_lens, _, out = _prep(scores, k, row_lens, None, out)
    val = torch.empty((R, k), dtype=torch.float32, device=scores.device) if values else None
    st = torch.zeros((R, len(STATS_FIELDS)), dtype=torch.int32, device=scores.device) if stats else None
    _check(_load().radix2_topk_batched_ex(_ptr(scores), stride, _ptr(row_lens), R, k, _ptr(out),
                                          _stream_ptr(stream), _ptr(val), _ptr(st)))
    return out, val, st


def _indexer_args(keys, row_set, q, w, row_lens):
    torch = _torch()
    if keys.dtype != torch.bfloat16 or keys.dim() != 3 or keys.shape[2] != 128 or not keys.is_contiguous() \
            or not keys.is_cuda:
        raise GvrError("keys must be a contiguous bf16 CUDA tensor [sets, n_max, 128]")
    R = row_set.shape[0]
    if row_set.dtype != torch.int32 or row_set.dim() != 1 or not row_set.is_cuda:
        raise GvrError("row_set must be int32 CUDA [R]")
    if q.dtype != torch.bfloat16 or tuple(q.shape) != (R, 64, 128) or not q.is_contiguous() or not q.is_cuda:
        raise GvrError("q must be a contiguous bf16 CUDA tensor [R, 64, 128]")
    if w.dtype != torch.float32 or tuple(w.shape) != (R, 64) or not w.is_contiguous() or not w.is_cuda:
        raise GvrError("w must be a contiguous fp32 CUDA tensor [R, 64]")
    if row_lens is not None and (row_lens.dtype != torch.int32 or tuple(row_lens.shape) != (R,) or not row_lens.is_cuda):
        raise GvrError("row_lens must be int32 CUDA [R]")
    return R, keys.shape[1]


def indexer_scores(keys, row_set, q, w, row_lens=None, out=None, stream=None):
    """DSA indexer scores (Eq. 1) on tensor cores: fp32 [R, n_max]."""
    torch = _torch()
    R, n_max = _indexer_args(keys, row_set, q, w, row_lens)
    if out is None:
        out = torch.zeros((R, n_max), dtype=torch.float32, device=keys.device)
    _check(_load().gvr_indexer_scores(_ptr(keys), n_max, _ptr(row_set), _ptr(row_lens), _ptr(q), _ptr(w), R,
                                      _ptr(out), out.stride(0), _stream_ptr(stream)))
    return out


def indexer_topk(keys, row_set, q, w, k: int = MAX_K, row_lens=None, prev=None, out=None, scratch=None,
                 stream=None):
    """Fused indexer -> GVR Top-K: the exact ordered Top-K of the indexer scores without
    writing them (scratch fp32 [R, n_max] is touched only for rows the lists cannot finish)."""
    torch = _torch()
    R, n_max = _indexer_args(keys, row_set, q, w, row_lens)
    if prev is not None and (prev.dtype != torch.int32 or tuple(prev.shape) != (R, k) or not prev.is_contiguous()):
        raise GvrError("prev must be a contiguous int32 CUDA tensor [R, k]")
    if out is None:
        out = torch.empty((R, k), dtype=torch.int32, device=keys.device)
    if scratch is None:
        scratch = torch.empty((R, n_max), dtype=torch.float32, device=keys.device)
    _check(_load().gvr_indexer_topk_batched(_ptr(keys), n_max, _ptr(row_set), _ptr(row_lens), _ptr(q), _ptr(w), R,
                                            _ptr(prev), k, _ptr(out), _ptr(scratch), _stream_ptr(stream)))
    return out


class Workspace:
    """Device buffers for the host-buffer entry point (gvr_topk_batched_host)."""

    def __init__(self, max_rows: int, row_stride: int, k: int = MAX_K):
        h = ctypes.c_void_p()
        _check(_load().gvr_workspace_create(max_rows, row_stride, k, ctypes.byref(h)))
        self._h, self.max_rows, self.row_stride, self.k = h, max_rows, row_stride, k

    def close(self):
        if self._h:
            _load().gvr_workspace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def topk_host(scores: np.ndarray, ws: Workspace, k: int = MAX_K, row_lens: np.ndarray | None = None,
              prev: np.ndarray | None = None, out: np.ndarray | None = None, stream=None) -> np.ndarray:
    """End-to-end entry: HOST fp32 scores [R, stride] (pinned recommended) -> HOST int32
    [R, k].  H2D copies, the GVR kernel and the D2H copy run inside the C call.
    row_lens [R] and prev [R, k] are converted to C-contiguous int32 when needed; out, if
    given, must already be a C-contiguous int32 [R, k] array (it is written in place)."""
    if not isinstance(scores, np.ndarray) or scores.dtype != np.float32 or scores.ndim != 2 \
            or not scores.flags.c_contiguous:
        raise GvrError("scores must be a C-contiguous fp32 [R, stride] array")
    R, stride = scores.shape
    if k != ws.k or stride != ws.row_stride or R > ws.max_rows:
        raise GvrError(f"workspace holds up to {ws.max_rows} rows of stride {ws.row_stride}, k={ws.k}")
    if out is None:
        out = np.empty((R, k), dtype=np.int32)
    elif not isinstance(out, np.ndarray) or out.dtype != np.int32 or out.shape != (R, k) \
            or not out.flags.c_contiguous:
        raise GvrError("out must be a C-contiguous int32 [R, k] array")
    if row_lens is not None:
        row_lens = np.ascontiguousarray(np.asarray(row_lens), dtype=np.int32)
        if row_lens.shape != (R,):
            raise GvrError("row_lens must have shape [R]")
    if prev is not None:
        prev = np.ascontiguousarray(np.asarray(prev), dtype=np.int32)
        if prev.shape != (R, k):
            raise GvrError("prev must have shape [R, k]")
    lp = None if row_lens is None else ctypes.c_void_p(row_lens.ctypes.data)
    pp = None if prev is None else ctypes.c_void_p(prev.ctypes.data)
    sp = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
    _check(_load().gvr_topk_batched_host(ctypes.c_void_p(scores.ctypes.data), stride, lp, R, pp, k,
                                         ctypes.c_void_p(out.ctypes.data), ws._h, sp))
    return out


def topk_host_ptr(scores_ptr: int, stride: int, R: int, ws: Workspace, k: int, out_ptr: int,
                  prev_ptr: int | None = None, lens_ptr: int | None = None, stream=None):
    """Same as topk_host on raw (pinned) host pointers."""
    sp = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
    _check(_load().gvr_topk_batched_host(ctypes.c_void_p(scores_ptr), stride,
                                         None if lens_ptr is None else ctypes.c_void_p(lens_ptr), R,
                                         None if prev_ptr is None else ctypes.c_void_p(prev_ptr), k,
                                         ctypes.c_void_p(out_ptr), ws._h, sp))
