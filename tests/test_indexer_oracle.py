"""Pins for the indexer oracle (oracle/indexer.py), CPU-only: Eq. 1 written out against
closed forms and an independent loop, and the tolerance checker against selections it
must accept and reject."""
import numpy as np
import pytest

from oracle import indexer as IX


def test_scores64_closed_forms():
    # one head, unit weight: ReLU of the dot product
    keys = np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, 2.0]])
    q = np.array([[2.0, 1.0]])
    assert IX.scores64(keys, q, np.array([1.0])).tolist() == [2.0, 1.0, 0.0]
    # two heads: sum of weighted ReLUs
    q2 = np.array([[1.0, 0.0], [0.0, -1.0]])
    assert IX.scores64(keys, q2, np.array([0.5, 3.0])).tolist() == [0.5, 0.0, 0.0]


def test_scores64_matches_a_loop():
    rng = np.random.default_rng(1)
    keys, q, w = rng.standard_normal((50, 16)), rng.standard_normal((4, 16)), rng.standard_normal(4)
    ref = [sum(w[j] * max(0.0, float(np.dot(q[j], keys[i]))) for j in range(4)) for i in range(50)]
    assert np.allclose(IX.scores64(keys, q, w), ref, rtol=0, atol=1e-12)


def test_check_topk_within_accepts_and_rejects():
    s = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    eps = np.full(5, 1e-9)
    IX.check_topk_within(np.array([0, 1, 2]), s, eps, 3)
    with pytest.raises(AssertionError):
        IX.check_topk_within(np.array([0, 1, 3]), s, eps, 3)  # misses 2
    with pytest.raises(AssertionError):
        IX.check_topk_within(np.array([1, 0, 2]), s, eps, 3)  # order
    # a near-tie inside the error bound may go either way
    s2 = np.array([5.0, 3.0, 3.0 + 1e-12, 1.0])
    IX.check_topk_within(np.array([0, 1]), s2, np.full(4, 1e-9), 2)
    IX.check_topk_within(np.array([0, 2]), s2, np.full(4, 1e-9), 2)
    IX.check_topk_within(np.array([1, 0, -1]), np.array([1.0, 2.0]), np.full(2, 1.0), 3)  # padding, order within eps


def test_error_bound_covers_fp32_evaluation():
    """An fp32 evaluation of Eq. 1 (a different accumulation order) stays within the bound."""
    rng = np.random.default_rng(2)
    keys = rng.standard_normal((200, 128)).astype(np.float32)
    q = rng.standard_normal((64, 128)).astype(np.float32)
    w = (rng.standard_normal(64) / 8).astype(np.float32)
    s32 = (w[None, :] * np.maximum(keys @ q.T, 0)).astype(np.float32).sum(axis=1, dtype=np.float32)
    err = np.abs(s32.astype(np.float64) - IX.scores64(keys, q, w))
    assert (err <= IX.score_error_bound(keys, q, w)).all()
