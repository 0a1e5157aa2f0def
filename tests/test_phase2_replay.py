"""Pins for the Phase 1-2 CPU replay (oracle/phase2_replay.py), CPU-only.

The replay is test infrastructure: it restates Phases 1-2 (DESIGN.md
R8-R12, R19, R34-R36) step by step so the GPU tests can compare the kernel's per-row
statistics (I, the Phase-2 exit, T_c) with it bit for bit.  Here it is pinned against
things other than itself: SPEC.md's worked Eq.-6 example, closed forms of the window
and of the sample layout, exact sums, and the invariants of the search.
"""
import math

import numpy as np
import pytest

from oracle import phase2_replay as P2

K = 2048


# --------------------------------------------------------------------------- Eq. 6
def test_secant_spec_example_undamped_and_damped():
    """(T_lo=0, f_lo=10000, T_hi=1, f_hi=0, f_target=4096) gives
    T_new = 0.5904 by direct substitution into Eq. 6, clamped to 0.5
    by first-iteration damping."""
    lo, hi = P2.key(0.0), P2.key(1.0)
    t = P2.secant_step(lo, 10000, hi, 0, np.float32(4096), damp=False, bisect=False)
    assert P2.unkey(t) == np.float32(0.5904)
    assert abs(float(P2.unkey(t)) - (10000 - 4096) / 10000) < 1e-7
    t = P2.secant_step(lo, 10000, hi, 0, np.float32(4096), damp=True, bisect=False)
    assert P2.unkey(t) == np.float32(0.5)


def test_secant_interpolates_linearly_between_anchors():
    """Eq. 6 on a bracket [2, 6] with counts 100 -> 20 and target 40: 2 + 60/80 * 4 = 5."""
    t = P2.secant_step(P2.key(2.0), 100, P2.key(6.0), 20, np.float32(40), damp=False, bisect=False)
    assert P2.unkey(t) == np.float32(5.0)
    # damping only caps fractions above 0.5
    t = P2.secant_step(P2.key(2.0), 100, P2.key(6.0), 20, np.float32(40), damp=True, bisect=False)
    assert P2.unkey(t) == np.float32(4.0)
    t = P2.secant_step(P2.key(2.0), 100, P2.key(6.0), 20, np.float32(80), damp=True, bisect=False)
    assert P2.unkey(t) == np.float32(3.0)  # fraction 0.25 is below the cap


def test_secant_bisection_fallbacks():
    """Bisection in key space (R11): when asked, when the float point is not strictly
    inside the bracket (float precision limit), or when the hi anchor is 2^32."""
    lo = P2.key(1.0)
    assert P2.secant_step(lo, 10, lo + 2, 0, np.float32(5), False, False) == lo + 1
    assert P2.secant_step(lo, 10, lo + 1000, 0, np.float32(5), False, True) == lo + 500
    assert P2.secant_step(0xFFFFFF00, 10, 1 << 32, 0, np.float32(5), False, False) == 0xFFFFFF00 + 0x80


# --------------------------------------------------------------------------- window
@pytest.mark.parametrize("n", [6017, 8192, 32768, 100_000, 131_072, 262_144])
def test_window_closed_form(n):
    """L = ceil(mu + 4.5 sqrt(mu)), mu = k S / n; H = L + ceil(L / 2); f_t = (L + H) / 2."""
    L, H, ft = P2.window(n, K)
    mu = K * 4096 / n
    assert L == math.ceil(mu + 4.5 * math.sqrt(mu))
    assert H == min(L + math.ceil(L / 2), 4096)
    assert float(ft) == (L + H) / 2


def test_window_cfg2_values():
    assert P2.window(100_000, K)[:2] == (126, 189)
    assert P2.window(131_072, K)[:2] == (100, 150)


# --------------------------------------------------------------------------- sample layout
def test_sample_positions_layout():
    """256 chunks of 16 contiguous floats, chunk c (thread c) at head + 16 floor(c nrun / 256)
    (R34)."""
    n, head = 100_003, 3
    pos = P2.sample_positions(n, head)
    assert pos.size == 4096 and len(np.unique(pos)) == 4096
    nrun = (4 * ((n - head) // 4)) // 16
    for c in (0, 1, 100, 255):
        start = head + 16 * ((c * nrun) // 256)
        assert list(pos[16 * c:16 * c + 16]) == list(range(start, start + 16))
    assert pos.max() < n and pos.min() == head
    gaps = np.diff(pos[::16])
    assert set(gaps) <= {16 * (nrun // 256), 16 * (nrun // 256 + 1)}


# --------------------------------------------------------------------------- Phase 1
def test_tree_sum_exact_on_integers():
    """Small integers sum exactly in fp32 in any order: the tree equals the exact sum."""
    rng = np.random.default_rng(1)
    v = rng.integers(-1000, 1000, size=(256, 8)).astype(np.float32)
    assert float(P2.tree_sum(v)) == float(v.astype(np.int64).sum())


def test_tree_sum_close_to_fsum():
    rng = np.random.default_rng(2)
    v = rng.standard_normal((256, 16)).astype(np.float32)
    assert abs(float(P2.tree_sum(v)) - math.fsum(v.astype(np.float64).ravel())) < 1e-3


def test_phase1_spec_example():
    """guessed values {1, 2, 3, 6} -> pmean 3.0, pmin 1.0, pmax 6.0."""
    x = np.zeros(10, np.float32)
    x[[1, 4, 6, 8]] = [1, 2, 3, 6]
    g = np.full(K, -1, np.int32)
    g[:4] = [1, 4, 6, 8]
    pmin, pmax, pmean, cnt = P2.phase1(x, g, K, 1)
    assert (P2.unkey(pmin), P2.unkey(pmax), pmean, cnt) == (1.0, 6.0, 3.0, 4)


def test_guessed_ranks_blocks():
    """R29: blocks of 8 consecutive ranks every 8 * stride ranks; stride 1 = all ranks."""
    assert list(P2.guessed_ranks(K, 1)) == list(range(2048))
    m = P2.guessed_ranks(K, 8)
    used = m[m < K]
    assert used.size == 256 and list(used[:10]) == [0, 1, 2, 3, 4, 5, 6, 7, 64, 65]
    assert used[-1] == 64 * 31 + 7


def test_phase1_ignores_out_of_range_and_strides():
    x = np.arange(1000, dtype=np.float32)
    g = np.full(K, -1, np.int32)
    g[0:8] = [5, -7, 2000, 9, 11, 1000, 13, 999]
    p = P2.phase1(x, g, K, 1)
    assert p[3] == 5 and P2.unkey(p[0]) == 5 and P2.unkey(p[1]) == 999
    assert p[2] == np.float32((5 + 9 + 11 + 13 + 999) / 5)
    # stride 2 reads ranks 0-7, 16-23, 32-39, ...: rank 8 is skipped, rank 16 is read
    g[8] = 500
    g[16] = 700
    assert P2.phase1(x, g, K, 1)[3] == 7
    p = P2.phase1(x, g, K, 2)
    assert p[3] == 6 and p[2] == np.float32((5 + 9 + 11 + 13 + 999 + 700) / 6)
    assert P2.phase1(x, np.full(K, -1, np.int32), K, 1) is None


# --------------------------------------------------------------------------- Phase 2
def _uniform_sample():
    """Sample keys of the values 0..4095 (one hit per value above T)."""
    return P2.keys(np.arange(4096, dtype=np.float32))


def test_phase2_t0_in_window_is_one_probe():
    """f(pmean) already in the window -> I = 1, converged at T0."""
    n = 100_000
    L, H, _ = P2.window(n, K)
    sk = _uniform_sample()
    t0 = np.float32(4096 - (L + H) // 2)  # hits(t0) = 4096 - t0 in [L, H]
    T, it, done, c = P2.phase2(sk, (P2.key(100.0), P2.key(4095.0), t0, K), n, K)
    assert (T, it, done, c) == (P2.key(t0), 1, P2.DONE_WINDOW, 4096 - int(t0))


def test_phase2_bracket_end_probe():
    """f(T0) below the window -> the second probe is pmin (Fig. 6's bracket end)."""
    n = 100_000
    L, H, _ = P2.window(n, K)
    sk = _uniform_sample()
    pmin = np.float32(4096 - L - 10)  # hits L + 10: inside the window
    T, it, done, c = P2.phase2(sk, (P2.key(pmin), P2.key(4095.0), np.float32(4090.0), K), n, K)
    assert (T, it, done, c) == (P2.key(pmin), 2, P2.DONE_WINDOW, L + 10)


def test_phase2_secant_converges_on_linear_counts():
    """On a uniform sample the count is linear in T, so after two probes outside the
    window the first (damped) secant step already lands in it or next to it."""
    n = 100_000
    L, H, _ = P2.window(n, K)
    sk = _uniform_sample()
    T, it, done, c = P2.phase2(sk, (P2.key(3000.0), P2.key(4095.0), np.float32(3500.0), K), n, K)
    assert done == P2.DONE_WINDOW and L <= c <= H and it <= 5
    assert c == int(np.count_nonzero(sk >= np.uint32(T)))


def test_phase2_ties_exit_takes_lo_anchor():
    """Two adjacent fp32 values only (no threshold with a count in the window): the
    anchors become adjacent keys -> DONE_TIES with the lo anchor (count above the window)."""
    n = 100_000
    v0 = np.float32(1.0)
    v1 = np.nextafter(v0, np.float32(np.inf))
    sk = P2.keys(np.r_[np.full(4000, v0, np.float32), np.full(96, v1, np.float32)])
    L, H, _ = P2.window(n, K)
    assert 96 < L  # 96 hits at v1 are below the window, 4096 at v0 above it
    T, it, done, c = P2.phase2(sk, (P2.key(v0), P2.key(v1), v1, K), n, K)
    assert (T, it, done, c) == (P2.key(v0), 1, P2.DONE_TIES, 4096)


def test_phase2_exhausted_exit_takes_sample_rank():
    """Two values far apart in key space: every probe lands on one side; after MAX_ITERS
    probes the exact finisher over the sample (R12) takes the key of rank ceil(f_t) —
    here the lower value (only 96 samples hold the upper one), whose hits are all 4096,
    above the window: its tie group spans the window, so the exit is a ties exit at that
    key (R37), and the filter path collects strictly above it."""
    n = 100_000
    sk = P2.keys(np.r_[np.zeros(4000, np.float32), np.ones(96, np.float32)])
    T, it, done, c = P2.phase2(sk, (P2.key(0.0), P2.key(1.0), np.float32(0.5), K), n, K)
    L, H, _ = P2.window(n, K)
    assert c > H
    assert done == P2.DONE_TIES and it == P2.MAX_ITERS
    assert T == P2.key(0.0) and c == 4096


def test_phase2_exhausted_rank_select_on_a_skewed_sample():
    """The finisher's key has exactly rank ceil(f_t) among distinct sample keys."""
    n = 100_000
    L, H, ft = P2.window(n, K)
    rank = (L + H + 1) // 2
    vals = np.exp(np.linspace(0, 30, 4096)).astype(np.float32)  # distinct, very skewed
    sk = P2.keys(vals)
    # force exhaustion: anchors far from the window with a probe budget of 0 secants
    T, it, done, c = P2.phase2(sk, None, n, K)
    if done == P2.DONE_EXHAUSTED:
        assert c == rank and T == int(np.sort(sk)[::-1][rank - 1])
    else:
        assert done == P2.DONE_WINDOW and L <= c <= H


def test_phase2_no_guess_uses_sample_statistics():
    rng = np.random.default_rng(3)
    x = rng.standard_normal(100_000).astype(np.float32)
    r = P2.replay_row(x, None, K)
    assert r["p1"][3] == 4096 and r["done"] == P2.DONE_WINDOW


def test_phase2_small_rows_collect_everything():
    r = P2.replay_row(np.ones(6016, np.float32), None, K)
    assert (r["Tc"], r["I"], r["done"]) == (0, 0, P2.DONE_ALL)


@pytest.mark.parametrize("seed", range(6))
def test_phase2_invariants_random_rows(seed):
    """On random rows: the exit is classified, a window exit has L <= hits <= H with hits
    recounted from the sample, I <= 12, and f(T_c) >= K on the full row."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(7000, 300_000))
    x = (rng.standard_normal(n) * rng.uniform(0.1, 10)).astype(np.float32)
    guess = rng.integers(0, n, K).astype(np.int32)
    head = int(rng.integers(0, 4))
    r = P2.replay_row(x, guess, K, head=head)
    sk = P2.keys(x[P2.sample_positions(n, head)])
    assert r["count"] == int(np.count_nonzero(sk >= np.uint32(r["Tc"])))
    assert 1 <= r["I"] <= P2.MAX_ITERS
    if r["done"] == P2.DONE_WINDOW:
        assert r["L"] <= r["count"] <= r["H"]
    assert int(np.count_nonzero(P2.keys(x) >= np.uint32(r["Tc"]))) >= K
