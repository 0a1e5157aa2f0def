"""Pins for the CPU oracle (oracle/), CPU-only.

The oracle is the definition of the result (exact ordered Top-K).  It is pinned here
against things other than itself: values printed in SPEC.md / hand-solved fixtures
(tests/golden/), closed forms, exhaustive brute force on tiny rows, a library sort in
the special case where both definitions provably coincide, and Lemma 1 of the paper.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _f(v):
    return float(v) if not isinstance(v, str) else float(v)


def _row(vals):
    return np.array([_f(v) for v in vals], dtype=np.float32)


def _load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


ALL_IMPLS = [oracle.topk, oracle.topk_rank, oracle.topk_numpy,
             lambda r, k: np.array(oracle.topk_bruteforce(r, k), dtype=np.int32)]


# --------------------------------------------------------------------------- golden
@pytest.mark.parametrize("case", _load("spec_examples.json")["topk_cases"],
                         ids=lambda c: c["citation"][:40])
def test_golden_topk(case):
    row = _row(case["row"])
    for impl in ALL_IMPLS:
        assert list(impl(row, case["k"])) == case["expect"], case["citation"]


@pytest.mark.parametrize("case", _load("spec_examples.json")["count_ge_cases"])
def test_golden_count_ge(case):
    assert oracle.count_ge(_row(case["row"]), case["t"]) == case["expect"]


@pytest.mark.parametrize("case", _load("spec_examples.json")["key_cases"])
def test_golden_key(case):
    x = _f(case["x"])
    assert oracle.sortable_key_c(x) == case["expect"]
    assert int(oracle.sortable_key(np.array([x], np.float32))[0]) == case["expect"]


def test_hand_k5_n10():
    fx = _load("hand_k5_n10.json")
    row = _row(fx["row"])
    for impl in ALL_IMPLS:
        assert list(impl(row, fx["k"])) == fx["expect"]


# --------------------------------------------------------------------------- key
def test_key_order_matches_float_order_special_values():
    vals = [-math.inf, -1e30, -1.0, -1e-40, -0.0, 0.0, 1e-40, 1.0, 1e30, math.inf]
    keys = [oracle.sortable_key_c(v) for v in vals]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


def test_key_monotone_random_pairs():
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2**32, size=200_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    a, b = x[::2], x[1::2]
    m = min(a.size, b.size)
    a, b = a[:m], b[:m]
    ka, kb = oracle.sortable_key(a), oracle.sortable_key(b)
    nz = ~((a == 0) & (b == 0))
    # for finite values that are not both zero: a < b  <=>  key(a) < key(b)
    assert np.array_equal((a < b)[nz], (ka < kb)[nz])
    # key is a bijection: distinct bit patterns give distinct keys
    assert np.array_equal(np.sort(oracle.sortable_key(x)).size, x.size)
    # C and numpy formulations agree
    for v in x[:2000]:
        assert oracle.sortable_key_c(float(v)) == int(oracle.sortable_key(np.array([v]))[0])


# --------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n,k", [(10, 5), (5000, 2048), (3000, 3000), (100, 1)])
def test_closed_forms(n, k):
    m = min(n, k)
    # all-equal row -> [0..k-1]
    assert list(oracle.topk(np.full(n, 3.5, np.float32), k)) == list(range(m)) + [-1] * (k - m)
    # x_i = i -> [n-1, n-2, ...]
    asc = np.arange(n, dtype=np.float32)
    assert list(oracle.topk(asc, k)) == list(range(n - 1, n - 1 - m, -1)) + [-1] * (k - m)
    # x_i = -i -> [0..k-1]
    assert list(oracle.topk(-asc, k)) == list(range(m)) + [-1] * (k - m)


def test_tie_fill_closed_forms():
    # 10,000 copies of 1.0, k=2048 -> indices 0..2047
    assert list(oracle.topk(np.ones(10_000, np.float32), 2048)) == list(range(2048))
    # one element above a 9,999-way tie -> it, then the first 2047 tied indices
    row = np.ones(10_000, np.float32)
    row[5000] = 2.0
    expect = [5000] + [i for i in range(10_000) if i != 5000][:2047]
    assert list(oracle.topk(row, 2048)) == expect


def test_empty_and_pad():
    assert list(oracle.topk(np.zeros(0, np.float32), 4)) == [-1, -1, -1, -1]
    assert list(oracle.topk_numpy(np.zeros(0, np.float32), 2)) == [-1, -1]


# --------------------------------------------------------------------------- brute force
def test_exhaustive_tiny_rows():
    """All rows over {-inf,-1,-0,+0,1,2,+inf}^n for n <= 5, every k <= n+1:
    the qsort oracle, the O(n^2) rank oracle, the numpy oracle and the pure-Python
    brute force (written independently from the rank definition) all agree."""
    alphabet = [-math.inf, -1.0, -0.0, 0.0, 1.0, 2.0, math.inf]
    checked = 0
    for n in range(0, 6):
        for combo in itertools.product(alphabet, repeat=n):
            row = np.array(combo, dtype=np.float32)
            k = n + 1
            ref = oracle.topk_bruteforce(row, k)
            assert list(oracle.topk(row, k)) == ref
            assert list(oracle.topk_rank(row, k)) == ref
            assert list(oracle.topk_numpy(row, k)) == ref
            # prefix property: the ordered Top-k for smaller k is a prefix
            for kk in range(0, k):
                assert list(oracle.topk(row, kk)) == ref[:kk]
            checked += 1
    assert checked == sum(7 ** n for n in range(6))


def test_brute_force_random_small():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        row = rng.integers(-4, 5, size=n).astype(np.float32)  # many ties
        k = int(rng.integers(1, n + 3))
        ref = oracle.topk_bruteforce(row, k)
        assert list(oracle.topk(row, k)) == ref
        assert list(oracle.topk_rank(row, k)) == ref


# --------------------------------------------------------------------------- library special case
def test_matches_torch_stable_sort_without_signed_zero():
    """On rows without -0/NaN, (key desc, idx asc) == a stable descending value sort."""
    import torch
    rng = np.random.default_rng(11)
    for n, k in [(8192, 2048), (100_000, 2048), (3000, 2048), (50, 7)]:
        row = rng.standard_normal(n).astype(np.float32)
        row[rng.integers(0, n, size=n // 10)] = row[0]  # inject ties
        row[row == 0] = 1.0
        t = torch.from_numpy(row)
        ref = torch.sort(t, descending=True, stable=True).indices[:k].numpy().astype(np.int32)
        assert np.array_equal(oracle.topk(row, k), ref)
        assert np.array_equal(oracle.topk_numpy(row, k), ref)


def test_topk_set_matches_torch_topk_when_kth_unique():
    """PAPER.md:848 correctness claim: index SET equals torch.topk's when the K-th value is unique."""
    import torch
    rng = np.random.default_rng(3)
    row = rng.permutation(131072).astype(np.float32)  # all distinct
    got = set(oracle.topk(row, 2048).tolist())
    ref = set(torch.topk(torch.from_numpy(row), 2048).indices.tolist())
    assert got == ref


# --------------------------------------------------------------------------- Lemma 1
def test_lemma1_containment():
    """PAPER.md:401-415 (Lemma 1): if K <= f(T) <= C then S* is a subset of {x >= T}."""
    rng = np.random.default_rng(5)
    K, C = 2048, 6144
    for trial in range(20):
        n = 20_000
        row = (rng.standard_normal(n) * (1 + trial)).astype(np.float32)
        s = np.sort(row)[::-1]
        top = set(oracle.topk(row, K).tolist())
        for t in (s[K - 1], s[(K + C) // 2], s[C - 1]):
            f = oracle.count_ge(row, t)
            assert K <= f <= C
            cand = set(np.nonzero(row >= t)[0].tolist())
            assert top <= cand


# --------------------------------------------------------------------------- batched
def test_batched_equals_per_row_with_ragged_lens():
    rng = np.random.default_rng(9)
    R, S, k = 17, 5000, 300
    scores = rng.standard_normal((R, S)).astype(np.float32)
    lens = rng.integers(0, S + 1, size=R).astype(np.int32)
    lens[0], lens[1] = 0, S
    out = oracle.topk_batched(scores, k, row_lens=lens, num_threads=4)
    for r in range(R):
        assert np.array_equal(out[r], oracle.topk(scores[r, :lens[r]], k))


def test_oracle_is_independent_of_product():
    """The oracle must not import or share code with the CUDA path."""
    import re
    here = os.path.dirname(oracle.__file__)
    bad = re.compile(r"^\s*(import\s+paper_2604_22312_b200|from\s+paper_2604_22312_b200|"
                     r"#\s*include\s*[<\"].*(csrc|gvr_topk|paper_2604))", re.M)
    for fn in os.listdir(here):
        if fn.endswith((".py", ".c", ".h")):
            with open(os.path.join(here, fn)) as fh:
                assert not bad.search(fh.read()), fn
