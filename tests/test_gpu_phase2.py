"""GPU: Phase 2 (the secant search of Eq. 6 over the row sample, R34-R36) and
the batch paths at the sizes and guess qualities the round-1 tests did not reach.

* The kernel's per-row Phase-2 statistics — T_c (as a key), I (probes), the exit kind
  and the sample hits at T_c — equal the CPU replay (oracle/phase2_replay.py) bit for bit,
  on every launch path (fused, cluster, batch filter, batch row).
* High-correlation decode rows (rho = 0.95 / 0.98 / 0.995, alpha up to ~0.8) on the
  filter path: exact, one HBM pass, no fixup rows.
* Filter-path batches at N = 131,072 (cfg5-shaped) and 262,144, a batch of massive ties
  that runs through the fixup kernel, the snap branch of Phase 4, MTP draft rows.
Every output is compared with the oracle element by element."""
import numpy as np
import pytest

import oracle
from oracle import phase2_replay as P2
import synth

pytestmark = pytest.mark.gpu
K = 2048
F = None  # STATS_FIELDS, set by the fixture


@pytest.fixture(scope="module")
def gvr(cuda_device):
    import __graft_entry__
    __graft_entry__.build()
    import paper_2604_22312_b200 as m
    global F
    F = m.STATS_FIELDS
    return m


def _col(st, name):
    return st[:, F.index(name)]


def _run(gvr, scores, lens, prev, k=K, opts=None):
    import torch
    idx, _, st = gvr.topk_ex(scores, k, row_lens=lens, prev=prev, values=False, options=opts)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), st.cpu().numpy()


def _assert_exact(got, ref, st=None):
    bad = np.argwhere((got != ref).any(axis=1))[:, 0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5].tolist()}" + (
        "" if st is None else f" stats {st[bad[:3]].tolist()}")


def _heads(R, stride):
    """Scalars before each row's first 16-byte boundary (torch bases are 16-B aligned)."""
    return [((16 - ((r * stride * 4) & 15)) & 15) >> 2 for r in range(R)]


def _assert_replay(host, lens, prev, st, k=K, stride_guess=8, rows=None, filter_path=False):
    """Kernel Phase-2 statistics == the CPU replay, row by row."""
    R, S = host.shape
    heads = _heads(R, S)
    rows = range(R) if rows is None else rows
    for r in rows:
        n = int(lens[r])
        if n <= k:
            continue
        rep = P2.replay_row(host[r, :n], None if prev is None else prev[r], k, head=heads[r], stride=stride_guess,
                            filter_path=filter_path)
        got = (int(_col(st, "tc_key")[r]) & 0xFFFFFFFF, int(_col(st, "secant_iters")[r]),
               int(_col(st, "phase2_exit")[r]), int(_col(st, "sample_count")[r]))
        exp = (rep["Tc"], rep["I"], rep["done"], rep["count"] if rep["done"] else 0)
        if rep["done"] == P2.DONE_ALL:
            exp = (0, 0, 0, 0)
        assert got == exp, f"row {r} n {n}: kernel {got} replay {exp}"


def _decode_batch(requests, layers, n, seed, rho=None, draft=1):
    import torch
    from bench import make_decode_batch
    b = make_decode_batch(requests, layers, n, torch.device("cuda:0"), seed=seed, draft=draft, rho=rho)
    torch.cuda.synchronize()
    return b


# ------------------------------------------------------------------ replay parity
@pytest.mark.parametrize("n", [8192, 40_000, 100_000, 262_144])
def test_phase2_stats_match_replay_fused_and_cluster(gvr, n):
    """Few rows (fused kernel, or a cluster per row when long): Phases 1-2 run inside the
    row's CTA; every CTA of a cluster computes the same T_c."""
    import torch
    rows, prevs = [], []
    for i, rho in enumerate((0.9, 0.0, 0.97)):
        p, c = synth.decode_pair(n, rho, seed=synth.splitmix64(2100, n, i))
        rows.append(c.numpy())
        prevs.append(oracle.topk(p.numpy(), K))
    rows.append(synth.dist_row("lognormal", n, seed=2101))
    prevs.append(np.full(K, -1, np.int32))  # no valid guess: sample statistics
    host = np.stack(rows)
    lens = np.full(len(rows), n, np.int32)
    prev = np.stack(prevs).astype(np.int32)
    dev = torch.device("cuda:0")
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev))
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    _assert_replay(host, lens, prev, st)


@pytest.mark.parametrize("path", [0, 1])
def test_phase2_stats_match_replay_batch_paths(gvr, path):
    """More than one wave (guess kernel + filter / row path), ragged lengths and strides
    that misalign rows, mixed guess kinds (prev step, random, adversarial, none)."""
    import torch
    rng = np.random.default_rng(2200 + path)
    R, S = 320, 70_001
    lens = rng.integers(3_000, S + 1, size=R).astype(np.int32)
    host = np.zeros((R, S), np.float32)
    prev = np.full((R, K), -1, np.int32)
    for r in range(R):
        n = int(lens[r])
        row = synth.dist_row(("normal", "lognormal", "uniform", "heavy_tail")[r % 4], n, seed=2201 + r)
        host[r, :n] = row
        kind = ("prev", "random", "adversarial", "none")[r % 4]
        noisy = row + 0.3 * rng.standard_normal(n).astype(np.float32) * np.float32(np.std(row) + 1e-6)
        g = synth.guess(kind, row, K, 2202 + r, prev_topk=oracle.topk(noisy, K))
        if g is not None:
            prev[r] = g
    dev = torch.device("cuda:0")
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev),
                   opts=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    _assert_replay(host, lens, prev, st, filter_path=path == 0)


# ------------------------------------------------------------------ high alpha
@pytest.mark.parametrize("rho", [0.95, 0.98, 0.995])
def test_high_alpha_filter_path_one_pass_no_fixup(gvr, rho):
    """Strongly correlated decode steps (alpha ~0.55-0.8, above the paper's 0.35-0.50 band,
    PAPER.md:275-277): Phase 2 keeps K <= f(T_c) on both sides of pmean, so every row of
    a 300-row N=100K filter-path batch is exact in one HBM pass with no fixup."""
    b = _decode_batch(5, 60, 100_000, seed=synth.splitmix64(2300, int(rho * 1000)), rho=rho)
    got, st = _run(gvr, b["scores"], b["row_lens"], b["prev"])
    host = b["scores"].cpu().numpy()
    lens = b["row_lens"].cpu().numpy()
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    assert (_col(st, "global_passes") == 1).all() and (_col(st, "done_kind") == 1).all(), st[:3].tolist()
    assert (_col(st, "phase2_exit") == 1).all()
    assert (_col(st, "buffer_count") >= K).all()
    # alpha really is high: the guess overlaps the exact Top-K
    prev = b["prev"].cpu().numpy()
    ref = oracle.topk_batched(host[:20], K, row_lens=lens[:20])
    alpha = np.mean([len(np.intersect1d(prev[r], ref[r])) / K for r in range(20)])
    assert alpha > 0.5
    _assert_replay(host, lens, prev, st, rows=range(0, 300, 37), filter_path=True)


# ------------------------------------------------------------------ sizes on the filter path
@pytest.mark.parametrize("n", [131_072, 262_144])
def test_filter_path_long_rows(gvr, n):
    """cfg5-shaped rows (N = 131,072) and N = 262,144 in 300-row batches: more than one
    wave, so the filter path (guess, filter, refine, fixup kernels) runs them."""
    b = _decode_batch(5, 60, n, seed=synth.splitmix64(2400, n))
    got, st = _run(gvr, b["scores"], b["row_lens"], b["prev"])
    host = b["scores"].cpu().numpy()
    lens = b["row_lens"].cpu().numpy()
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    assert (_col(st, "global_passes") == 1).all()
    assert (_col(st, "cluster") == 1).all()


def test_filter_path_mtp_draft_rows(gvr):
    """cfg4-shaped rows: 4 draft tokens per request, each one more decode step past the
    shared guess (alpha decays along the draft), N + j keys."""
    b = _decode_batch(16, 5, 100_000, seed=2450, draft=4)
    got, st = _run(gvr, b["scores"], b["row_lens"], b["prev"])
    host = b["scores"].cpu().numpy()
    lens = b["row_lens"].cpu().numpy()
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    assert (_col(st, "global_passes") == 1).all()


def test_massive_ties_batch_through_fixup(gvr):
    """300 rows of all-equal / few-distinct / 90%-tied values: the refine kernel cannot
    finish them from their lists (crowded K-th bin), the fixup kernel streams them again
    and fills the ties in index order; exact."""
    import torch
    R, n = 300, 50_000
    kinds = ("all_equal", "few_distinct", "ties90")
    rows = [synth.dist_row(kinds[r % 3], n - (r % 7), seed=2500 + r) for r in range(R)]
    S = n
    host = np.zeros((R, S), np.float32)
    lens = np.array([r.size for r in rows], np.int32)
    for r, row in enumerate(rows):
        host[r, :row.size] = row
    prev = np.stack([synth.guess("random", rows[r], K, 2501 + r) for r in range(R)]).astype(np.int32)
    dev = torch.device("cuda:0")
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev))
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    assert (_col(st, "done_kind") == 2).sum() > 0  # tie fill ran


def test_ties90_exhausted_becomes_ties_exit(gvr):
    """488 rows of N = 100K with 90% of the values tied at 0.25 (synth.dist_row ties90) on
    the filter path: rows whose sample cannot reach the window end at the tie key; that
    key's sample count is above the window, so the exit is a ties exit (R37) and the row is
    collected strictly above the tie instead of taking the whole tie group into its list.
    Phase-2 statistics equal the CPU replay row by row, no row needs the fixup, exact."""
    import torch
    R, n = 488, 100_000
    host = np.stack([synth.dist_row("ties90", n, seed=9000 + r) for r in range(R)]).astype(np.float32)
    lens = np.full(R, n, np.int32)
    prev = np.stack([synth.guess("random", host[r], K, 9001 + r) for r in range(R)]).astype(np.int32)
    dev = torch.device("cuda:0")
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev))
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    _assert_replay(host, lens, prev, st, filter_path=True, rows=range(0, R, 3))
    assert (_col(st, "phase2_exit") == P2.DONE_TIES).sum() > 0
    assert (_col(st, "phase2_exit") == P2.DONE_EXHAUSTED).sum() == 0
    assert (_col(st, "global_passes") == 1).all()
    assert (_col(st, "cand_count") < 8 * K).all()


def test_snap_branch_runs(gvr):
    """A tie group of 300 at the row maximum crowds one bin above the K-th one, so the
    sorted-bin shortcut (R28) is refused and Phase 4's snap iterations
    find T*: snap_iters > 0, exact."""
    import torch
    rows = []
    for i in range(3):
        row = synth.dist_row("normal", 60_000, seed=2600 + i)
        row[np.random.default_rng(i).choice(60_000, 300, replace=False)] = np.float32(50.0)
        rows.append(row)
    host = np.stack(rows)
    lens = np.full(3, 60_000, np.int32)
    prev = np.stack([synth.guess("random", r, K, 2601) for r in rows]).astype(np.int32)
    dev = torch.device("cuda:0")
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev),
                   opts=gvr.GvrOptions(float("nan"), 0, 1, 0))  # one CTA per row (the row kernel)
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)
    assert (_col(st, "snap_iters") > 0).all(), st.tolist()


# ------------------------------------------------------------------ same-geometry radix
@pytest.mark.parametrize("n,R", [(100_000, 300), (262_144, 8), (20_001, 5), (9_000, 400)])
def test_radix2_baseline_exact(gvr, n, R):
    """The same-geometry radix baseline (histogram pass on the half digit + the GVR filter /
    refine kernels) equals the oracle at any batch size, including long rows split across
    CTAs and ragged lengths."""
    import torch
    rng = np.random.default_rng(2700 + n)
    lens = rng.integers(max(1, n // 2), n + 1, size=R).astype(np.int32)
    lens[0] = n
    if R > 3:
        lens[1], lens[2] = 1000, 2048  # trivial rows
    host = np.zeros((R, n), np.float32)
    for r in range(R):
        host[r, :lens[r]] = synth.dist_row(("normal", "lognormal", "uniform", "heavy_tail")[r % 4], int(lens[r]),
                                           seed=2701 + r)
    dev = torch.device("cuda:0")
    idx, val, st = gvr.radix2_topk_ex(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev))
    torch.cuda.synchronize()
    _assert_exact(idx.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens), st.cpu().numpy())


def test_radix2_baseline_ties_and_decode_rows(gvr):
    import torch
    b = _decode_batch(2, 61, 100_000, seed=2800)
    host = b["scores"].cpu().numpy()
    lens = b["row_lens"].cpu().numpy()
    host[3] = 1.0  # massive ties: the list overflows, the fixup kernel finishes the row
    host[5, ::3] = 7.0
    idx = gvr.radix2_topk(torch.from_numpy(host).cuda(), K, row_lens=b["row_lens"])
    torch.cuda.synchronize()
    _assert_exact(idx.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))


# ------------------------------------------------------------------ ultra-long rows
@pytest.mark.parametrize("n", [1 << 20, 1 << 22])
def test_ultra_long_single_rows(gvr, n):
    """Rows far beyond any CTA's or cluster's shared memory (1M and 4M elements): the
    cluster kernel streams its slices (the row is never resident); exact."""
    import torch
    rows = [synth.dist_row(kind, n, seed=2900 + i) for i, kind in enumerate(("normal", "lognormal"))]
    host = np.stack(rows)
    lens = np.full(2, n, np.int32)
    dev = torch.device("cuda:0")
    prev = np.stack([synth.guess("random", r, K, 2901) for r in rows]).astype(np.int32)
    got, st = _run(gvr, torch.from_numpy(host).to(dev), torch.from_numpy(lens).to(dev), torch.from_numpy(prev).to(dev))
    _assert_exact(got, oracle.topk_batched(host, K, row_lens=lens), st)


def test_ultra_long_batch_filter_path(gvr):
    """300 rows of 512K elements (more than one wave: the filter path, each row split over
    several filter CTAs)."""
    import torch
    R, n = 300, 1 << 19
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3000)
    s = torch.randn((R, n), generator=g, device=dev)
    prev = torch.randint(0, n, (R, K), generator=g, device=dev, dtype=torch.int32)
    lens = torch.full((R,), n, dtype=torch.int32, device=dev)
    got, st = _run(gvr, s, lens, prev)
    _assert_exact(got, oracle.topk_batched(s.cpu().numpy(), K), st)
    assert (_col(st, "global_passes") == 1).all()


def test_fixup_kernel_short_lists(gvr):
    """A Phase-2 window aimed below the K-th value (window_z = -8) leaves every filter-path
    list short: the refine hands all 300 rows to the fixup kernel, which streams each once
    more at the second-pass threshold (R30, skipping the known-short first stream)."""
    import torch
    R, n = 300, 9_000
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3100)
    s = torch.randn((R, n), generator=g, device=dev)
    prev = torch.randint(0, n, (R, K), generator=g, device=dev, dtype=torch.int32)
    lens = torch.full((R,), n, dtype=torch.int32, device=dev)
    got, st = _run(gvr, s, lens, prev, opts=gvr.GvrOptions(-8.0, 0, 0, 0, 0))
    _assert_exact(got, oracle.topk_batched(s.cpu().numpy(), K), st)
    assert (_col(st, "global_passes") == 2).all(), st[:3].tolist()


# ------------------------------------------------------------------ indexer (f3)
def _indexer_inputs(sets, rows_per_set, n, seed, rho=0.9):
    """bf16 key sets from the Eq.-1 generator (RoPE'd keys) and per-row bf16 queries / fp32
    weights: row j of set s is the query of draft j (one more AR step each)."""
    import torch
    dev = torch.device("cuda:0")
    keys, qs, ws, row_set, lay_prev = [], [], [], [], []
    for si in range(sets):
        lay = synth.IndexerLayer(n, rho, synth.splitmix64(seed, si), dev)
        keys.append(lay.keys[:n].to(torch.bfloat16))
        for j in range(rows_per_set):
            if j:
                lay.step()
            qs.append(lay.query(n).to(torch.bfloat16))
            ws.append(lay.w.clone())
            row_set.append(si)
    return (torch.stack(keys).contiguous(), torch.tensor(row_set, dtype=torch.int32, device=dev),
            torch.stack(qs).contiguous(), torch.stack(ws).float().contiguous())


def test_indexer_scores_match_eq1(gvr):
    """Tensor-core indexer scores (bf16 inputs, fp32 accumulation) equal Eq. 1 evaluated in
    fp64 from the same bf16 inputs within the fp32 rounding bound; ragged lengths."""
    import torch
    from oracle import indexer as IX
    keys, row_set, q, w = _indexer_inputs(2, 3, 5_000, seed=3200)
    lens = torch.tensor([5_000, 4_999, 77, 4_096, 1, 3_333], dtype=torch.int32, device="cuda:0")
    out = gvr.indexer_scores(keys, row_set, q, w, row_lens=lens)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    kh, qh, wh = keys.float().cpu().numpy(), q.float().cpu().numpy(), w.cpu().numpy()
    for r in range(6):
        n = int(lens[r])
        s64 = IX.scores64(kh[int(row_set[r]), :n], qh[r], wh[r])
        eps = IX.score_error_bound(kh[int(row_set[r]), :n], qh[r], wh[r])
        assert (np.abs(o[r, :n] - s64) <= eps).all(), (r, float(np.abs(o[r, :n] - s64).max()), float(eps.min()))
        assert (o[r, n:] == 0).all()


@pytest.mark.parametrize("sets,rows_per_set,n", [(4, 1, 20_000), (80, 4, 9_000), (3, 2, 100_000)])
def test_indexer_topk_fused(gvr, sets, rows_per_set, n):
    """Fused indexer -> Top-K (f3): (a) bit-identical to the unfused path (the same scores
    materialised by gvr_indexer_scores, then gvr_topk_batched) — fusion changes nothing;
    (b) a valid ordered Top-K of Eq. 1 evaluated in fp64 from the same bf16 inputs, within
    the fp32 rounding bound.  Batches of one wave and of more (the filter path), MTP rows
    sharing a key set, ragged lengths including a row of <= k keys."""
    import torch
    from oracle import indexer as IX
    keys, row_set, q, w = _indexer_inputs(sets, rows_per_set, n, seed=3300 + n)
    R = row_set.shape[0]
    rng = np.random.default_rng(3301)
    lens_np = rng.integers(n // 2, n + 1, size=R).astype(np.int32)
    lens_np[0] = n
    if R > 2:
        lens_np[1] = 1500  # <= k: materialised by the fixup
    lens = torch.from_numpy(lens_np).cuda()
    prev = torch.from_numpy(np.stack([rng.integers(0, n, K) for _ in range(R)]).astype(np.int32)).cuda()
    fused = gvr.indexer_topk(keys, row_set, q, w, K, row_lens=lens, prev=prev)
    sc = gvr.indexer_scores(keys, row_set, q, w, row_lens=lens)
    unfused = gvr.topk(sc, K, row_lens=lens, prev=prev)
    torch.cuda.synchronize()
    fo, uo = fused.cpu().numpy(), unfused.cpu().numpy()
    _assert_exact(fo, uo)
    kh, qh, wh = keys.float().cpu().numpy(), q.float().cpu().numpy(), w.cpu().numpy()
    for r in range(0, R, max(1, R // 6)):
        m = int(lens_np[r])
        kk = kh[int(row_set[r]), :m]
        IX.check_topk_within(fo[r], IX.scores64(kk, qh[r], wh[r]), IX.score_error_bound(kk, qh[r], wh[r]), K)
