"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

The DSA indexer scores of PAPER.md Eq. 1 (lines 78-81) in fp64, and the tolerance rules
for checking a Top-K selected from fp32 scores computed on the GPU:

    I_t[i] = sum_j W_j * ReLU(Q_j . K_i)

from the same bf16 (or any) inputs, evaluated in float64 with numpy (a plain matrix
product, then ReLU, then the weighted head sum — Eq. 1 written out).  The GPU accumulates
in fp32 in its own order, so its scores differ from these by at most the fp32 rounding
bound `score_error_bound` (a dot product of m terms accumulated in fp32 carries at most
~m * 2^-24 of the sum of the absolute terms); a selection is accepted when it is a valid
Top-K under that bound (`check_topk_within`).  Parity pin: tests/test_indexer_oracle.py.
"""
from __future__ import annotations

import numpy as np


def scores64(keys: np.ndarray, q: np.ndarray, w: np.ndarray) -> np.ndarray:
    """keys [n, d], q [h, d], w [h] (any float dtype) -> fp64 scores [n] (Eq. 1)."""
    k = np.asarray(keys, dtype=np.float64)
    qq = np.asarray(q, dtype=np.float64)
    ww = np.asarray(w, dtype=np.float64)
    logits = qq @ k.T                       # [h, n]: Q_j . K_i
    return ww @ np.maximum(logits, 0.0)     # sum_j W_j ReLU(.)


def score_error_bound(keys: np.ndarray, q: np.ndarray, w: np.ndarray, rel: float = 2.0 ** -17) -> np.ndarray:
    """Per-key bound on |fp32 score - fp64 score|: rel * sum_j |W_j| sum_d |Q_jd K_id|
    (rel = 2^-17 covers a 128-term fp32 dot product plus the 64-term weighted sum, each
    term's rounding at most 2^-24 of the running absolute sum, with margin)."""
    k = np.abs(np.asarray(keys, dtype=np.float64))
    qq = np.abs(np.asarray(q, dtype=np.float64))
    ww = np.abs(np.asarray(w, dtype=np.float64))
    return rel * (ww @ (qq @ k.T)) + 1e-30


def check_topk_within(sel: np.ndarray, s64: np.ndarray, eps: np.ndarray, k: int) -> None:
    """A selection (k indices in output order) is a valid ordered Top-K of the true scores
    s64 up to the per-key error eps: (1) k distinct in-range indices; (2) every key whose
    score exceeds the k-th true score by more than 2 eps is selected, and every selected key
    is within 2 eps of it or above; (3) consecutive outputs are ordered up to their eps."""
    n = s64.size
    m = min(k, n)
    sel = np.asarray(sel, dtype=np.int64)
    assert (sel[m:] == -1).all(), "padding"
    s = sel[:m]
    assert len(np.unique(s)) == m and s.min() >= 0 and s.max() < n, "distinct in-range indices"
    kth = np.sort(s64)[::-1][m - 1]
    e = float(eps.max())
    must = np.nonzero(s64 > kth + 2 * e)[0]
    assert np.isin(must, s).all(), f"{np.setdiff1d(must, s).size} keys clearly above the K-th value missing"
    assert (s64[s] >= kth - 2 * e).all(), "a selected key is clearly below the K-th value"
    d = s64[s[:-1]] - s64[s[1:]]
    assert (d >= -(eps[s[:-1]] + eps[s[1:]])).all(), "output order"
