"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

Step-by-step CPU replay of Phases 1-2 of GVR as the batch path runs them (PAPER.md
Sec. 4.2.1-4.2.2; R8-R11, R19, R34-R36): the previous step's
Top-K positions give pmin / pmax / pmean (Eq. 4), and the secant search of Eq. 6 looks
for a threshold T whose count lies in a target window — counting over a fixed row
sample instead of the whole row (R34).  This is the "kernel-faithful replay of the
Phase-2 control flow" of PAPER.md:576-586 / 1672-1683: every fp32 operation is written
out in the order and rounding the kernel uses (explicit round-to-nearest, no fused
multiply-add), so the replay reproduces the kernel's I (secant_iters), the Phase-2 exit
kind and the threshold T_c bit for bit.  It is written from the paper and DESIGN.md,
not from the CUDA source, and shares no code with it.

Parity: the threshold statistics are not part of the result contract (the output is
the exact Top-K whatever T_c is, Lemma 1); they are pinned here by
closed-form cases in tests/test_phase2_replay.py (Eq. 6 substitution of SPEC.md's
worked example, damping, bisection, window arithmetic) and compared with the kernel's
per-row stats in the GPU tests.
"""
from __future__ import annotations

import numpy as np

# Constants of the batch path's Phase 2 (R34-R36).
SAMPLE_CHUNKS = 256        # 16-float chunks per row sample (one per guess-kernel thread)
CHUNK = 16                 # floats per chunk (one 64-byte read)
S = SAMPLE_CHUNKS * CHUNK  # 4096 sample values
RUN = 16                   # floats per contiguous sample run (R34): one chunk
NRUN = S // RUN            # 256 runs per row sample
Z = np.float32(4.5)        # window lower edge: mu + Z sqrt(mu) sample hits (R35)
MAX_SECANT = 8             # secant steps before pure bisection (R11)
MAX_ITERS = 12             # count evaluations before the Phase-2 fallback (R12)
CAP_ALL = 6016             # rows with n <= CAP_ALL collect every element (T_c = -inf)
GUESS_THREADS = 256        # the reduction tree of the guess kernel (pmean)
GUESS_SLOTS = 8            # guessed positions per thread (2048 / 256)
DONE_WINDOW, DONE_TIES, DONE_EXHAUSTED, DONE_ALL = 1, 2, 3, 0

f32 = np.float32


def key(x) -> int:
    """Sortable uint32 key of one fp32 value."""
    u = int(np.array([x], dtype=np.float32).view(np.uint32)[0])
    return (~u & 0xFFFFFFFF) if (u & 0x80000000) else (u | 0x80000000)


def unkey(k: int) -> np.float32:
    u = (k ^ 0x80000000) if (k & 0x80000000) else (~k & 0xFFFFFFFF)
    return np.array([u], dtype=np.uint32).view(np.float32)[0]


def keys(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return np.where(u & np.uint32(0x80000000), ~u, u | np.uint32(0x80000000)).astype(np.uint32)


def sample_positions(n: int, head: int) -> np.ndarray:
    """Row positions of the sample, in guess-kernel thread order (R34): 256 runs of
    16 contiguous floats, run g (thread g's chunk) at head + 16 * floor(g * nrun / 256) with
    nrun = floor(body / 16) runs of the 16-byte aligned body (head = scalars before the
    first 16-byte boundary)."""
    body = 4 * ((n - head) // 4)
    nrun = body // RUN
    c = np.arange(SAMPLE_CHUNKS, dtype=np.int64)
    starts = head + RUN * (((c // (RUN // CHUNK)) * nrun) // NRUN) + CHUNK * (c % (RUN // CHUNK))
    return (starts[:, None] + np.arange(CHUNK)[None, :]).ravel()


def window(n: int, k: int, z=Z):
    """Target window [L, H] and target f_t in sample hits (R35): mu = k S / n expected
    hits at the K-th value; L = ceil(mu + z sqrt(mu)) (at least 1, at most S),
    H = L + ceil(L / 2) (at most S), f_t = (L + H) / 2 — the sample image of the paper's
    [K, C] window and f_target = (K + C) / 2."""
    mu = f32(f32(k * S) / f32(n))
    lo = f32(mu + f32(f32(z) * np.sqrt(mu, dtype=np.float32)))
    L = min(max(int(np.ceil(lo)), 1), S)
    H = min(L + (L + 1) // 2, S)
    ft = f32(f32(L + H) * f32(0.5))
    return L, H, ft


def tree_sum(vals: np.ndarray) -> np.float32:
    """fp32 sum in the guess kernel's order: thread t (of 256) adds its values
    sequentially (vals[t, j], j = 0, 1, ...), each warp sums its 32 lanes with an
    xor-butterfly (offsets 16, 8, 4, 2, 1), then warp 0 does the same over the 8 warp
    sums (lanes >= 8 contribute 0)."""
    vals = np.asarray(vals, dtype=np.float32).reshape(GUESS_THREADS, -1)
    per = np.zeros(GUESS_THREADS, dtype=np.float32)
    for j in range(vals.shape[1]):
        per = (per + vals[:, j]).astype(np.float32)

    def butterfly(v):
        v = v.astype(np.float32).copy()
        for o in (16, 8, 4, 2, 1):
            v = (v + v[np.arange(32) ^ o]).astype(np.float32)
        return v[0]

    warps = np.array([butterfly(per[32 * w:32 * (w + 1)]) for w in range(GUESS_THREADS // 32)],
                     dtype=np.float32)
    lanes = np.zeros(32, dtype=np.float32)
    lanes[:warps.size] = warps
    return butterfly(lanes)


def guessed_ranks(k: int, stride: int) -> np.ndarray:
    """Ranks of the guess list used by Phase 1 (R29), slot i = 0..2047 (thread i % 256,
    register i // 256): m_i = 8 stride floor(i / 8) + i % 8, used while m_i < k —
    blocks of 8 consecutive ranks every 8 stride ranks; stride 1 = every rank."""
    i = np.arange(GUESS_THREADS * GUESS_SLOTS, dtype=np.int64)
    return 8 * stride * (i >> 3) + (i & 7)


def phase1(x: np.ndarray, guess, k: int, stride: int):
    """pmin, pmax (keys) and pmean (Eq. 4) over the valid guessed
    positions q = guess[m_i] (guessed_ranks); positions outside [0, n) are ignored (R7).
    Returns (pmin_key, pmax_key, pmean, count), or None when no position is valid."""
    n = x.size
    if guess is None:
        return None
    g = np.asarray(guess, dtype=np.int64)
    m = guessed_ranks(k, stride)
    pos = np.full(m.size, -1, dtype=np.int64)
    use = m < k
    pos[use] = g[m[use]]
    ok = (pos >= 0) & (pos < n)
    vals = np.where(ok, x[np.clip(pos, 0, n - 1)], np.float32(0)).astype(np.float32)
    if not ok.any():
        return None
    kk = keys(vals[ok])
    # slot i = t + 256 j belongs to thread t; invalid slots add +0
    s = tree_sum(vals.reshape(GUESS_SLOTS, GUESS_THREADS).T)
    cnt = int(ok.sum())
    pmean = f32(s / f32(cnt))
    return int(kk.min()), int(kk.max()), pmean, cnt


def secant_step(klo: int, clo: int, khi: int, chi: int, ft: np.float32, damp: bool, bisect: bool) -> int:
    """Eq. 6 in value space between the anchors (klo, clo > target)
    and (khi, chi < target), khi exclusive (may be 2^32); first-step damping caps the
    fraction at 0.5; bisection in key space when the point is not
    strictly inside (klo, khi), not finite, or bisect is set (R11, R19)."""
    if not bisect and khi <= 0xFFFFFFFF:
        flo, fhi = unkey(klo), unkey(khi)
        with np.errstate(all="ignore"):
            frac = f32(f32(f32(clo) - ft) / f32(clo - chi))
            if damp:
                frac = min(frac, f32(0.5))
            tf = f32(flo + f32(frac * f32(fhi - flo)))
        if np.isfinite(tf):
            kt = key(tf)
            if klo < kt < khi:
                return kt
    return klo + ((khi - klo) >> 1)


def phase2(sample_keys: np.ndarray, p1, n: int, k: int, z=Z, max_secant: int = MAX_SECANT):
    """Phase 2 over the sample (PAPER.md:527-570 with R8-R12, R34-R36).

    Anchors are exact for the sample (SPEC.md's virtual anchors, R8): lo = (min key, S),
    hi = (max key + 1, 0).  The first probe is T0 = pmean (Fig. 6)
    when it lies strictly inside; every probe counts the sample keys >= T (the kernel's
    blockCountGE over the sample), accepts a count in [L, H], else moves the anchor on
    its side and takes the Eq. 6 step toward f_t (damped on the first secant step;
    bisection after MAX_SECANT steps or when the bracket is too narrow for a float
    point).  Before the first secant step it probes T0 = pmean and then the Phase-1
    bracket end on the far side of the window.  Exits: DONE_WINDOW (T_c = T), DONE_TIES
    (adjacent anchors: no key in the window — a tie group spans it; T_c = the lo anchor,
    whose count is above the window), DONE_EXHAUSTED (MAX_ITERS probes; T_c = the sample
    key of rank ceil(f_t), the exact finisher over the sample — DONE_TIES instead when that
    key's count is above the window: its tie group spans the window, R37).
    Returns (T_c key, I = probes, done, count at T_c)."""
    L, H, ft = window(n, k, z)
    sk = np.asarray(sample_keys, dtype=np.uint32)
    klo, clo = int(sk.min()), S
    khi, chi = int(sk.max()) + 1, 0
    it = 0

    def probe(T):
        nonlocal klo, clo, khi, chi, it
        c = int(np.count_nonzero(sk >= np.uint32(T)))
        it += 1
        if L <= c <= H:
            return c
        if c > H:
            klo, clo = T, c
        else:
            khi, chi = T, c
        return -c - 1  # not in the window

    # T0 = pmean (Fig. 6), then the Phase-1 bracket end on the far
    # side of the window (pmin when f(T0) < L, pmax when f(T0) > H; Fig. 6's bracket
    # [pmin, pmax]) — each probed only if strictly inside the current anchors
    if p1 is not None and np.isfinite(p1[2]):
        t0 = key(p1[2])
        if klo < t0 < khi:
            r = probe(t0)
            if r >= 0:
                return t0, it, DONE_WINDOW, r
            t1 = p1[0] if -r - 1 < L else p1[1]
            if klo < t1 < khi:
                r = probe(t1)
                if r >= 0:
                    return t1, it, DONE_WINDOW, r
    first_secant = True
    secants = 0
    while True:
        if khi - klo < 2:
            return klo, it, DONE_TIES, clo
        if it >= MAX_ITERS:
            # the exact finisher over the sample (R12): the key of rank ceil(f_t)
            rank = (L + H + 1) // 2
            T = int(np.sort(sk)[::-1][rank - 1])
            c = int(np.count_nonzero(sk >= np.uint32(T)))
            # a key whose tie group reaches past the window: a ties exit at it (R37)
            return T, it, DONE_TIES if c > H else DONE_EXHAUSTED, c
        T = secant_step(klo, clo, khi, chi, ft, first_secant, secants >= max_secant)
        first_secant = False
        secants += 1
        r = probe(T)
        if r >= 0:
            return T, it, DONE_WINDOW, r


def replay_row(x: np.ndarray, guess, k: int, head: int = 0, stride: int = 8, z=Z, max_secant: int = MAX_SECANT,
               filter_path: bool = False):
    """Phases 1-2 of one row as the guess kernel runs them (head: the row's scalars before
    its first 16-byte boundary; stride: the guess stride, every row).  Returns a
    dict with the collect threshold key Tc, I, done (Phase-2 exit), window (L, H), the
    sample count at Tc and the Phase-1 tuple p1 = (pmin key, pmax key, pmean, count)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.size
    if n <= CAP_ALL:
        return dict(Tc=0, I=0, done=DONE_ALL, L=0, H=0, count=0)
    p1 = phase1(x, guess, k, stride)
    sv = x[sample_positions(n, head)]
    sk = keys(sv)
    if p1 is None:
        # no valid guess: Phase-1 statistics over the row sample instead (SPEC.md:287,
        # R7); thread t holds chunk t's 16 values
        p1 = (int(sk.min()), int(sk.max()), f32(tree_sum(sv.reshape(SAMPLE_CHUNKS, CHUNK)) / f32(S)), S)
    Tc, it, done, c = phase2(sk, p1, n, k, z, max_secant)
    L, H, _ = window(n, k, z)
    tie = Tc if done == DONE_TIES else 0
    if filter_path and done == DONE_TIES and Tc < 0xFFFFFFFF:
        Tc += 1  # the batch filter path collects strictly above the tied key (R37)
    return dict(Tc=Tc, I=it, done=done, L=L, H=H, count=c, p1=p1, tie=tie)
