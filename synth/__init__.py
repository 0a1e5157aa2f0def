"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module generates *inputs only*: DSA indexer score rows (Eq. 1, lines
78-81) built from random RoPE'd queries/keys, guess index sets of several kinds, and
value distributions for edge-case tests.  It holds none of the Top-K method's
arithmetic (no thresholds, counts, secant steps or selection); both the CUDA path and
the CPU oracle consume what it produces.  Recipe and calibration: DESIGN.md "Inputs".

Sources restated (not copied) from PAPER.md:
  * Eq. 1 indexer: I_t = sum_j W_j * ReLU(Q_{t,j} K^T), h = 64 heads, d_i = 128
    (PAPER.md:78-81, 204, 821-822).
  * YaRN inverse frequencies for the 64 RoPE dims, base 1e4, scale 40, original
    context 4096, beta_fast 32, beta_slow 1 (App. E 1539-1549).
  * Split-half rotation layout.
  * App. E single-head synthetic rows with amplitude Am = 0.1.
  * Eq. 3 static RoPE prior: the K largest g(Delta).
"""
from __future__ import annotations

import math
import zlib

import numpy as np
import torch

BASE_SEED = 260422312
MASK64 = (1 << 64) - 1


def splitmix64(*parts: int) -> int:
    """Deterministic 64-bit seed from integer parts (splitmix64 finaliser chain)."""
    z = 0
    for p in parts:
        z = (z + 0x9E3779B97F4A7C15 + (int(p) & MASK64)) & MASK64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        z = z ^ (z >> 31)
    return z & ((1 << 63) - 1)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


# ----------------------------------------------------------------------------- RoPE
def yarn_inv_freq(dim: int = 64, base: float = 10000.0, scale: float = 40.0,
                  orig_ctx: int = 4096, beta_fast: float = 32.0, beta_slow: float = 1.0) -> torch.Tensor:
    """YaRN-interpolated inverse frequencies (restating PAPER.md App. E 1539-1549).

    theta_i = base^(-2i/dim).  Dimensions whose wavelength is short relative to the
    original context keep theta_i ("extrapolation"); long-wavelength dimensions use
    theta_i/scale ("interpolation"); a linear ramp between the correction dims
    lo = floor(d(beta_fast)) and hi = ceil(d(beta_slow)) blends the two, where
    d(beta) = dim * ln(orig_ctx / (2*pi*beta)) / (2 ln base).
    """
    i = torch.arange(0, dim, 2, dtype=torch.float64)
    theta = base ** (-i / dim)

    def corr_dim(beta):
        return dim * math.log(orig_ctx / (beta * 2 * math.pi)) / (2 * math.log(base))

    lo = max(math.floor(corr_dim(beta_fast)), 0)
    hi = min(math.ceil(corr_dim(beta_slow)), dim - 1)
    span = max(hi - lo, 1e-3)
    ramp = ((torch.arange(dim // 2, dtype=torch.float64) - lo) / span).clamp(0.0, 1.0)
    return (theta / scale * ramp + theta * (1.0 - ramp)).to(torch.float32)


def rope_rotate(x: torch.Tensor, pos: torch.Tensor, inv_freq: torch.Tensor) -> torch.Tensor:
    """Rotate the last dim of x (size 2*len(inv_freq)) by angle pos*theta, split-half layout:
    even dims a, odd dims b -> cat(a cos - b sin, b cos + a sin)."""
    ang = pos.to(torch.float32)[..., None] * inv_freq.to(x.device)
    c, s = torch.cos(ang), torch.sin(ang)
    a, b = x[..., 0::2], x[..., 1::2]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1)


def g_delta(n: int, inv_freq: torch.Tensor | None = None) -> np.ndarray:
    """g(Delta) = 2 sum_i cos(Delta theta_i), Delta = 0..n-1 (Eq. 2, 314-319)."""
    if inv_freq is None:
        inv_freq = yarn_inv_freq()
    th = inv_freq.to(torch.float64).numpy()
    d = np.arange(n, dtype=np.float64)
    return 2.0 * np.cos(np.outer(d, th)).sum(axis=1)


def static_prior(n: int, k: int = 2048, query_pos: int | None = None) -> np.ndarray:
    """Eq. 3 static prior: the k positions m whose relative distance
    Delta = |query_pos - m| to the query has the largest g(Delta).  The query sits at the
    newest position n - 1 by default (the Eq.-1 decode rows, IndexerLayer); the App.-E
    listing rotates it at position 0 (appendix_e_row: query_pos=0).  Input generation
    only."""
    qp = n - 1 if query_pos is None else int(query_pos)
    m = np.arange(n, dtype=np.int64)
    g = g_delta(n)[np.abs(qp - m)]
    kk = min(k, n)
    pos = np.argsort(-g, kind="stable")[:kk].astype(np.int32)
    out = np.full(k, -1, dtype=np.int32)
    out[:kk] = pos
    return out


# ----------------------------------------------------------------------------- Eq. 1 rows
class IndexerLayer:
    """One (request, layer) of the synthetic DSA indexer (Eq. 1).

    Keys K ~ N(0,1) in R^{n x 128} are frozen; the first ``d_rope`` dims of every key at
    position m are rotated by m (YaRN RoPE).  Queries Q_t in R^{64 x 128} and head
    weights W_t ~ N(0, 1/64) evolve as AR(1) processes with coefficient ``rho``
    (Q_t = rho Q_{t-1} + sqrt(1-rho^2) xi_t).  The step-t query is rotated at the
    newest position (row length - 1).  Scores are fp32 with TF32 disabled.
    """

    def __init__(self, n_max: int, rho: float, seed: int, device="cpu",
                 heads: int = 64, dim: int = 128, d_rope: int = 64):
        self.n_max, self.rho, self.heads, self.dim, self.d_rope = n_max, rho, heads, dim, d_rope
        self.device = torch.device(device)
        self.inv_freq = yarn_inv_freq(d_rope).to(self.device)
        g = _gen(splitmix64(seed, 1), self.device)
        keys = torch.randn(n_max, dim, generator=g, device=self.device)
        pos = torch.arange(n_max, device=self.device)
        keys[:, :d_rope] = rope_rotate(keys[:, :d_rope], pos, self.inv_freq)
        self.keys = keys
        self._g = _gen(splitmix64(seed, 2), self.device)
        self.q = torch.randn(heads, dim, generator=self._g, device=self.device)
        self.w = torch.randn(heads, generator=self._g, device=self.device) / math.sqrt(heads)

    def step(self):
        """Advance the AR(1) query/weight state by one decode step."""
        r = self.rho
        s = math.sqrt(max(0.0, 1.0 - r * r))
        self.q = r * self.q + s * torch.randn(self.heads, self.dim, generator=self._g, device=self.device)
        self.w = r * self.w + s * torch.randn(self.heads, generator=self._g, device=self.device) / math.sqrt(self.heads)

    def query(self, n: int) -> torch.Tensor:
        """The step's indexer query Q_t [heads, dim], RoPE'd at the newest position n - 1."""
        q = self.q.clone()
        q[:, :self.d_rope] = rope_rotate(q[:, :self.d_rope],
                                         torch.full((self.heads,), n - 1, device=self.device),
                                         self.inv_freq)
        return q

    def scores(self, n: int) -> torch.Tensor:
        """Eq. 1 score row over the first n keys for the current query state (fp32)."""
        assert 0 < n <= self.n_max
        q = self.q.clone()
        q[:, :self.d_rope] = rope_rotate(q[:, :self.d_rope],
                                         torch.full((self.heads,), n - 1, device=self.device),
                                         self.inv_freq)
        prev_tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            logits = torch.relu(q @ self.keys[:n].T)  # [heads, n]
            row = (self.w[None, :] @ logits).squeeze(0)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev_tf32
        return row.contiguous()


def layer_rho(layer: int, seed: int) -> float:
    """Per-layer AR(1) coefficient: layers 0-1 uncorrelated (alpha ~ 1-3%, like DSV3.2
    L0-1); layers >= 2 rho ~ U[0.88, 0.93] (alpha ~ 0.35-0.50, like
    L20-60).  Calibration in DESIGN.md."""
    if layer < 2:
        return 0.0
    u = (splitmix64(seed, 77, layer) % 10_000) / 10_000.0
    return 0.88 + 0.05 * u


def decode_pair(n: int, rho: float, seed: int, device="cpu", steps_between: int = 1):
    """Scores of two consecutive decode steps of one indexer layer.

    Returns (prev_row [n-1], cur_row [n]) as fp32 tensors: the previous step sees n-1
    keys, the current step one more (the KV cache grows by one token per step)."""
    lay = IndexerLayer(n, rho, seed, device)
    prev = lay.scores(n - 1)
    for _ in range(steps_between):
        lay.step()
    cur = lay.scores(n)
    return prev, cur


def appendix_e_row(n: int, seed: int, am: float = 0.1, d_rope: int = 64, device="cpu") -> torch.Tensor:
    """App. E single-head synthetic row: q, k ~ 1 + Am N(0,1), both
    RoPE'd on d_rope dims, query at position 0 (as in the listing)."""
    dev = torch.device(device)
    g = _gen(splitmix64(seed, 3), dev)
    inv = yarn_inv_freq(d_rope).to(dev)
    q = 1.0 + am * torch.randn(1, d_rope, generator=g, device=dev)
    k = 1.0 + am * torch.randn(n, d_rope, generator=g, device=dev)
    qr = rope_rotate(q, torch.zeros(1, device=dev), inv)
    kr = rope_rotate(k, torch.arange(n, device=dev), inv)
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return (qr @ kr.T).squeeze(0).contiguous()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32


# ----------------------------------------------------------------------------- test distributions
DISTRIBUTIONS = ("uniform", "normal", "lognormal", "heavy_tail", "ties90", "all_equal",
                 "few_distinct", "signed_zero_mix", "with_inf", "sorted_asc", "sorted_desc",
                 "negative", "tiny_range", "beta", "weibull", "logistic")
# the score shapes fitted to the real DSV3.2 layers (Table 7):
# beta (bounded, peaked: L21/L40/L41), weibull (right-skewed: L22/L60), logistic
# (heavy-tailed: L1), lognormal (heterogeneous: L0)
TABLE7_SHAPES = ("beta", "weibull", "logistic", "lognormal")


def dist_row(kind: str, n: int, seed: int) -> np.ndarray:
    """fp32 row of length n with the named value distribution (edge-case tests)."""
    rng = np.random.default_rng(splitmix64(seed, 5, zlib.crc32(kind.encode())))
    if kind == "uniform":
        x = rng.random(n)
    elif kind == "normal":
        x = rng.standard_normal(n)
    elif kind == "lognormal":
        x = rng.lognormal(0.0, 1.5, n)
    elif kind == "heavy_tail":
        x = rng.standard_t(1.5, n)
    elif kind == "ties90":
        x = rng.standard_normal(n)
        x[rng.random(n) < 0.9] = 0.25
    elif kind == "all_equal":
        x = np.full(n, -1.75)
    elif kind == "few_distinct":
        x = rng.integers(0, 5, n).astype(np.float64)
    elif kind == "signed_zero_mix":
        x = np.where(rng.random(n) < 0.5, 0.0, -0.0)
        x[rng.random(n) < 0.02] = 1.0
        x[rng.random(n) < 0.02] = -1.0
    elif kind == "with_inf":
        x = rng.standard_normal(n)
        x[rng.random(n) < 0.01] = np.inf
        x[rng.random(n) < 0.01] = -np.inf
    elif kind == "sorted_asc":
        x = np.sort(rng.standard_normal(n))
    elif kind == "sorted_desc":
        x = np.sort(rng.standard_normal(n))[::-1]
    elif kind == "negative":
        x = -rng.lognormal(1.0, 0.5, n)
    elif kind == "tiny_range":
        x = 1.0 + rng.integers(0, 3000, n) * np.finfo(np.float32).eps
    elif kind == "beta":
        x = rng.beta(2.0, 5.0, n)
    elif kind == "weibull":
        x = rng.weibull(1.5, n)
    elif kind == "logistic":
        x = rng.logistic(0.0, 1.0, n)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(x.astype(np.float32))


GUESS_KINDS = ("prev", "static", "random", "adversarial", "duplicates", "out_of_range",
               "all_minus1", "none")


def guess(kind: str, row: np.ndarray, k: int, seed: int, prev_topk: np.ndarray | None = None):
    """Guess index set of the named kind for ``row`` (None for kind 'none').

    'prev' needs the previous step's Top-K passed in as ``prev_topk``; 'adversarial'
    picks the k positions of the *lowest* values (a worst case for the threshold guess)."""
    n = row.size
    rng = np.random.default_rng(splitmix64(seed, 9, zlib.crc32(kind.encode())))
    if kind == "none":
        return None
    if kind == "prev":
        assert prev_topk is not None
        return np.ascontiguousarray(prev_topk.astype(np.int32))
    if kind == "static":
        return static_prior(n, k)
    if kind == "random":
        return rng.integers(0, max(n, 1), k).astype(np.int32)
    if kind == "adversarial":
        order = np.argsort(row, kind="stable")[:k].astype(np.int32)
        out = np.full(k, -1, np.int32)
        out[:order.size] = order
        return out
    if kind == "duplicates":
        return np.full(k, int(rng.integers(0, max(n, 1))), np.int32)
    if kind == "out_of_range":
        g = rng.integers(-3 * n - 5, 3 * n + 5, k).astype(np.int64)
        return np.clip(g, -2**31, 2**31 - 1).astype(np.int32)
    if kind == "all_minus1":
        return np.full(k, -1, np.int32)
    raise ValueError(kind)
