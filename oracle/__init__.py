"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU reference for the GVR exact Top-K hot path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  It never imports the
product package ``paper_2604_22312_b200`` and the product never imports it; the
two share no code (the only shared module is the seeded input generator
``synth/``, which holds none of the method's arithmetic).

What is computed (PAPER.md = /root/reference/PAPER.md):

* ``topk`` / ``topk_batched`` — the exact Top-K of a row (PAPER.md:385-388,
  Sec. 4.1), ordered by score descending then index ascending (BASELINE.json
  north_star), ``-1`` padded when n < k (R5).
  Scores are ordered by the sortable FP32 key,
  so +0 ranks above -0 and NaNs sit beyond +/-Inf (R3, R4).
  Backed by ``topk_oracle.c`` (qsort of (key, idx) pairs).
* ``topk_numpy`` — the same definition with ``numpy.lexsort`` as the sort step.
* ``topk_bruteforce`` — the rank definition in pure Python (tiny rows only).
* ``count_ge`` — the counting function f(T) = |{i : x_i >= T}|.

Pins: every function above is checked in ``tests/test_oracle.py`` against values
fixed by the paper/SPEC examples (``tests/golden/``), closed forms, exhaustive brute
force on tiny rows, and ``torch.sort(stable=True)`` on rows where the two
definitions provably coincide.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "topk_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile topk_oracle.c into liboracle.so with the host C compiler."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_sortable_key.restype = ctypes.c_uint32
            lib.oracle_sortable_key.argtypes = [ctypes.c_float]
            for name in ("oracle_topk_row", "oracle_topk_rank_row"):
                fn = getattr(lib, name)
                fn.restype = ctypes.c_int
                fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
            lib.oracle_topk_batched.restype = ctypes.c_int
            lib.oracle_topk_batched.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                                ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                                ctypes.c_int32]
            _lib = lib
    return _lib


def _as_f32(row) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(row, dtype=np.float32))
    return a


def sortable_key(x) -> np.ndarray:
    """Sortable uint32 key of fp32 values, numpy formulation."""
    u = _as_f32(x).view(np.uint32)
    neg = (u & np.uint32(0x80000000)) != 0
    return np.where(neg, ~u, u | np.uint32(0x80000000)).astype(np.uint32)


def sortable_key_c(x: float) -> int:
    """Sortable key of one fp32 value, C formulation."""
    return int(_load().oracle_sortable_key(ctypes.c_float(x)))


def topk(row, k: int) -> np.ndarray:
    """Exact ordered Top-K of one row via the C oracle (qsort of (key, idx))."""
    a = _as_f32(row).ravel()
    out = np.empty(k, dtype=np.int32)
    rc = _load().oracle_topk_row(a.ctypes.data, a.size, k, out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_topk_row failed")
    return out


def topk_rank(row, k: int) -> np.ndarray:
    """Exact ordered Top-K of one row via the C O(n^2) rank formulation."""
    a = _as_f32(row).ravel()
    out = np.empty(k, dtype=np.int32)
    rc = _load().oracle_topk_rank_row(a.ctypes.data, a.size, k, out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_topk_rank_row failed")
    return out


def topk_batched(scores: np.ndarray, k: int, row_lens=None, num_threads: int | None = None) -> np.ndarray:
    """Exact ordered Top-K of every row of ``scores`` [R, stride] (host, fp32)."""
    s = np.ascontiguousarray(np.asarray(scores, dtype=np.float32))
    if s.ndim != 2:
        raise ValueError("scores must be 2-D")
    R, stride = s.shape
    out = np.empty((R, k), dtype=np.int32)
    lens_ptr = None
    if row_lens is not None:
        lens = np.ascontiguousarray(np.asarray(row_lens, dtype=np.int32))
        if lens.shape != (R,):
            raise ValueError("row_lens must have shape [R]")
        lens_ptr = lens.ctypes.data
    if num_threads is None:
        num_threads = os.cpu_count() or 1
    rc = _load().oracle_topk_batched(s.ctypes.data, stride, lens_ptr, R, k, out.ctypes.data,
                                     int(num_threads))
    if rc != 0:
        raise ValueError("oracle_topk_batched failed")
    return out


def topk_numpy(row, k: int) -> np.ndarray:
    """Same definition with numpy.lexsort as the sort step (key desc, idx asc)."""
    key = sortable_key(row).ravel()
    n = key.size
    idx = np.arange(n, dtype=np.int64)
    order = np.lexsort((idx, ~key))  # last key is primary: ~key ascending == key descending
    out = np.full(k, -1, dtype=np.int32)
    m = min(k, n)
    out[:m] = order[:m]
    return out


def topk_bruteforce(row, k: int) -> list:
    """Rank definition in pure Python (tiny rows): rank_i = #{j : j precedes i}."""
    keys = [int(v) for v in sortable_key(row).ravel()]
    n = len(keys)
    out = [-1] * k
    for i in range(n):
        rank = sum(1 for j in range(n) if keys[j] > keys[i] or (keys[j] == keys[i] and j < i))
        if rank < k:
            out[rank] = i
    return out


def count_ge(row, t: float) -> int:
    """f(T) = |{i : x_i >= T}|, in float comparison."""
    a = _as_f32(row).ravel()
    return int(np.count_nonzero(a >= np.float32(t)))
