"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, bit-exact (integer index output; BASELINE.json: "bit-exactly, both as an index
set and in order").  Every input is seeded and synthetic (synth/)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
K = 2048


@pytest.fixture(scope="module")
def gvr(cuda_device):
    import __graft_entry__
    __graft_entry__.build()
    import paper_2604_22312_b200 as m
    return m


def _pack(rows, stride=None):
    S = max([r.size for r in rows] + [1]) if stride is None else stride
    host = np.zeros((len(rows), S), np.float32)
    lens = np.array([r.size for r in rows], np.int32)
    for i, r in enumerate(rows):
        host[i, :r.size] = r
    return host, lens


def _run(gvr, host, lens, k, prev=None, impl="gvr", values=False):
    import torch
    dev = torch.device("cuda:0")
    s = torch.from_numpy(host).to(dev)
    l = torch.from_numpy(lens).to(dev)
    if impl == "gvr":
        p = None if prev is None else torch.from_numpy(np.ascontiguousarray(prev, np.int32)).to(dev)
        idx, val, st = gvr.topk_ex(s, k, row_lens=l, prev=p)
    else:
        idx, val, st = gvr.radix_topk_ex(s, k, row_lens=l)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), val.cpu().numpy(), st.cpu().numpy()


def _check(gvr, rows, k=K, prevs=None, stride=None, impls=("gvr", "radix")):
    host, lens = _pack(rows, stride)
    ref = oracle.topk_batched(host, k, row_lens=lens)
    prev = None
    if prevs is not None:
        prev = np.stack([np.asarray(p, np.int32) if p is not None else np.full(k, -1, np.int32)
                         for p in prevs])
    for impl in impls:
        got, val, st = _run(gvr, host, lens, k, prev, impl)
        if not np.array_equal(got, ref):
            bad = np.argwhere((got != ref).any(axis=1))[:, 0]
            r = int(bad[0])
            j = int(np.argwhere(got[r] != ref[r])[0][0])
            raise AssertionError(f"{impl}: {len(bad)} rows differ; row {r} len {lens[r]} first diff at "
                                 f"{j}: got {got[r, j]} ref {ref[r, j]}; stats {st[r].tolist()}")
        # values are x[idx] (bit-exact), 0 for padding
        for r in range(len(rows)):
            m = min(k, lens[r])
            exp = np.zeros(k, np.float32)
            exp[:m] = host[r, ref[r, :m]]
            assert np.array_equal(val[r].view(np.uint32), exp.view(np.uint32)), (impl, r)
    return ref


# ------------------------------------------------------------------ Eq. 1 decode rows
@pytest.mark.parametrize("n,rho", [(8192, 0.9), (32768, 0.9), (100_000, 0.9), (100_000, 0.0),
                                   (131_072, 0.93), (262_144, 0.9)])
def test_indexer_rows_prev_step_guess(gvr, n, rho):
    rows, prevs = [], []
    for i in range(3):
        prev_row, cur = synth.decode_pair(n, rho, seed=synth.splitmix64(synth.BASE_SEED, n, i))
        rows.append(cur.numpy())
        prevs.append(oracle.topk(prev_row.numpy(), K))
    _check(gvr, rows, prevs=prevs)


def test_appendix_e_rows_static_prior(gvr):
    rows, prevs = [], []
    for n in (8192, 16384, 70_690):
        rows.append(synth.appendix_e_row(n, seed=n).numpy())
        prevs.append(synth.static_prior(n, K, query_pos=0))  # the App.-E query sits at position 0
    _check(gvr, rows, prevs=prevs)


# ------------------------------------------------------------------ sizes / edges
SIZES = [1, 2, 5, 10, K - 1, K, K + 1, 6143, 6144, 6145, 12287, 12288, 12289, 8192, 8193,
         20_001, 65_537, 100_003]


@pytest.mark.parametrize("n", SIZES)
def test_sizes_normal(gvr, n):
    rows = [synth.dist_row("normal", n, seed=n), synth.dist_row("uniform", n, seed=n + 1)]
    _check(gvr, rows, prevs=[synth.guess("random", rows[0], K, 1), None])


@pytest.mark.parametrize("k", [1, 2, 7, 64, 100, 1000, 2047])
def test_small_k(gvr, k):
    rows = [synth.dist_row("normal", n, seed=n + k) for n in (1, 3, k, k + 1, 5000, 40_000)]
    prevs = [synth.guess("random", r, k, 3) for r in rows]
    _check(gvr, rows, k=k, prevs=prevs)


@pytest.mark.parametrize("kind", synth.DISTRIBUTIONS)
@pytest.mark.parametrize("n", [3000, 30_000, 150_000])
def test_distributions(gvr, kind, n):
    row = synth.dist_row(kind, n, seed=7)
    rows = [row, row.copy()]
    prevs = [synth.guess("adversarial", row, K, 2), synth.guess("random", row, K, 2)]
    _check(gvr, rows, prevs=prevs)


def test_nan_ordering_is_deterministic(gvr):
    row = synth.dist_row("normal", 50_000, seed=3)
    row[::997] = np.nan
    row[5] = -np.nan
    _check(gvr, [row], prevs=[synth.guess("random", row, K, 1)])


# ------------------------------------------------------------------ layout
@pytest.mark.parametrize("stride_pad", [1, 2, 3, 5])
def test_misaligned_row_stride(gvr, stride_pad):
    n = 30_001
    rows = [synth.dist_row("normal", n, seed=s) for s in range(5)]
    _check(gvr, rows, stride=n + stride_pad, prevs=[synth.guess("random", r, K, 4) for r in rows])


def test_ragged_row_lens(gvr):
    rng = np.random.default_rng(5)
    rows = [synth.dist_row("lognormal", int(m), seed=int(m)) for m in rng.integers(0, 70_000, 24)]
    rows += [np.zeros(0, np.float32), synth.dist_row("normal", 1, seed=1)]
    _check(gvr, rows, prevs=[synth.guess("random", r, K, 5) if r.size else None for r in rows])


# ------------------------------------------------------------------ guess robustness
@pytest.mark.parametrize("n", [9000, 100_000])
def test_output_independent_of_guess(gvr, n):
    import torch
    prev_row, cur = synth.decode_pair(n, 0.9, seed=11)
    cur = cur.numpy()
    prev_topk = oracle.topk(prev_row.numpy(), K)
    host, lens = _pack([cur])
    ref = oracle.topk_batched(host, K, row_lens=lens)
    outs = []
    for kind in synth.GUESS_KINDS:
        g = synth.guess(kind, cur, K, 9, prev_topk=prev_topk)
        got, _, st = _run(gvr, host, lens, K, None if g is None else g[None, :])
        assert np.array_equal(got, ref), (kind, st.tolist())
        outs.append(got.tobytes())
    assert len(set(outs)) == 1


def test_in_place_prev_equals_out(gvr):
    import torch
    n = 100_000
    rows, prevs = [], []
    for i in range(4):
        p, c = synth.decode_pair(n, 0.9, seed=100 + i)
        rows.append(c.numpy())
        prevs.append(oracle.topk(p.numpy(), K))
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, K, row_lens=lens)
    dev = torch.device("cuda:0")
    buf = torch.from_numpy(np.stack(prevs)).to(dev)
    gvr.topk(torch.from_numpy(host).to(dev), K, prev=buf, out=buf)
    torch.cuda.synchronize()
    assert np.array_equal(buf.cpu().numpy(), ref)


# ------------------------------------------------------------------ full-size config
@pytest.mark.parametrize("path", [0, 1])
def test_full_size_cfg2_batch(gvr, path):
    """BASELINE.json configs[1]: 8 requests x 61 layers at N=100K, prev-step guesses,
    in the launch configuration bench.py times (one call over all 488 rows), on the
    filter path (0, the default) and the row path (1)."""
    import torch
    from bench import make_decode_batch
    dev = torch.device("cuda:0")
    batch = make_decode_batch(8, 61, 100_000, dev, seed=synth.BASE_SEED, draft=1)
    torch.cuda.synchronize()
    host = batch["scores"].cpu().numpy()
    lens = batch["row_lens"].cpu().numpy()
    ref = oracle.topk_batched(host, K, row_lens=lens)
    out = gvr.topk(batch["scores"], K, row_lens=batch["row_lens"], prev=batch["prev"],
                   options=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
    rad = gvr.radix_topk(batch["scores"], K, row_lens=batch["row_lens"])
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    assert np.array_equal(rad.cpu().numpy(), ref)


def test_stats_sanity(gvr):
    rows, prevs = [], []
    for i in range(6):
        p, c = synth.decode_pair(100_000, 0.9 if i else 0.0, seed=200 + i)
        rows.append(c.numpy())
        prevs.append(oracle.topk(p.numpy(), K))
    host, lens = _pack(rows)
    _, _, st = _run(gvr, host, lens, K, np.stack(prevs))
    for s in st:
        secant, snap, cand, done, passes, raises, bufcnt, cluster, p2exit, scount, tc, _ = s.tolist()
        assert done == 1 and passes == 1  # converged, one HBM pass
        assert 1 <= secant <= 12 and K <= cand <= 6144 and K <= bufcnt <= 6144
        assert cluster >= 1 and p2exit == 1 and 1 <= scount <= 4096


def test_host_buffer_entry_point(gvr):
    n, R = 50_000, 6
    rows = [synth.dist_row("normal", n, seed=300 + i) for i in range(R)]
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, K, row_lens=lens)
    ws = gvr.Workspace(R, n, K)
    prev = np.stack([synth.guess("random", r, K, 8) for r in rows])
    got = gvr.topk_host(host, ws, K, prev=prev)
    assert np.array_equal(got, ref)
    got2 = gvr.topk_host(host, ws, K, row_lens=lens)
    assert np.array_equal(got2, ref)
    ws.close()


# ------------------------------------------------------------------ launch plumbing
def _decode_rows(R, n=60_000, seed=400):
    rows, prevs = [], []
    for i in range(R):
        p, c = synth.decode_pair(n, 0.9 if i % 3 else 0.0, seed=seed + i)
        rows.append(c.numpy())
        prevs.append(oracle.topk(p.numpy(), K))
    host, lens = _pack(rows)
    return host, lens, np.stack(prevs)


def test_cuda_graph_capture_and_replay(gvr):
    """The GVR call (guess kernel, streaming kernel and their hand-off scratch) captures
    into a CUDA graph; replays on new inputs written into the same buffers are exact."""
    import torch
    dev = torch.device("cuda:0")
    host_a, lens, prev_a = _decode_rows(5, seed=410)
    host_b, _, prev_b = _decode_rows(5, seed=420)
    s = torch.from_numpy(host_a).to(dev)
    l = torch.from_numpy(lens).to(dev)
    p = torch.from_numpy(prev_a).to(dev)
    out = torch.empty((5, K), dtype=torch.int32, device=dev)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        gvr.topk(s, K, row_lens=l, prev=p, out=out)  # warm-up on the capture stream (sizes its scratch)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gvr.topk(s, K, row_lens=l, prev=p, out=out)
    for host, prev in ((host_a, prev_a), (host_b, prev_b)):
        s.copy_(torch.from_numpy(host))
        p.copy_(torch.from_numpy(prev))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))


def test_concurrent_streams(gvr):
    """Two streams running GVR concurrently each keep their own hand-off scratch."""
    import torch
    dev = torch.device("cuda:0")
    jobs = [_decode_rows(7, seed=430), _decode_rows(9, n=80_000, seed=440)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for (host, lens, prev), st in zip(jobs, streams):
        with torch.cuda.stream(st):
            s = torch.from_numpy(host).to(dev, non_blocking=False)
            l = torch.from_numpy(lens).to(dev)
            p = torch.from_numpy(prev).to(dev)
            res = []
            for _ in range(3):
                res.append(gvr.topk(s, K, row_lens=l, prev=p))
            outs.append(res)
    torch.cuda.synchronize()
    for (host, lens, _), res in zip(jobs, outs):
        ref = oracle.topk_batched(host, K, row_lens=lens)
        for o in res:
            assert np.array_equal(o.cpu().numpy(), ref)


def test_events_entry_point(gvr):
    import torch
    dev = torch.device("cuda:0")
    host, lens, prev = _decode_rows(4, seed=450)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = gvr.topk_events(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                          prev=torch.from_numpy(prev).to(dev), events=evs)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))
    assert evs[0].elapsed_time(evs[1]) >= 0 and evs[1].elapsed_time(evs[2]) > 0
    assert evs[2].elapsed_time(evs[3]) >= 0


def test_events_entry_point_filter_path(gvr):
    """More than one wave: the four events bracket the guess, filter and refine kernels."""
    import torch
    dev = torch.device("cuda:0")
    host, lens, prev = _decode_rows(300, n=12_000, seed=460)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = gvr.topk_events(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                          prev=torch.from_numpy(prev).to(dev), events=evs)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))
    assert all(evs[i].elapsed_time(evs[i + 1]) > 0 for i in range(3))


# ------------------------------------------------------------------ cluster per row
def _run_cluster(gvr, host, lens, prev, G):
    import torch
    dev = torch.device("cuda:0")
    p = None if prev is None else torch.from_numpy(np.ascontiguousarray(prev, np.int32)).to(dev)
    idx, val, st = gvr.topk_ex(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev), prev=p,
                               options=gvr.GvrOptions(float("nan"), 0, G, 0))
    torch.cuda.synchronize()
    return idx.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("n", [2047, 6000, 20_001, 100_000, 262_144])
def test_cluster_rows(gvr, G, n):
    """A cluster of G CTAs per row (slices merged into the leader through DSMEM) gives
    the oracle's output, for good (rho 0.9) and poor (rho 0) previous-step guesses."""
    rows, prevs = [], []
    for i, rho in enumerate((0.9, 0.0, 0.92)):
        p, c = synth.decode_pair(n, rho, seed=500 + 7 * i + n % 97)
        rows.append(c.numpy())
        prevs.append(oracle.topk(p.numpy(), K))
    host, lens = _pack(rows)
    got, st = _run_cluster(gvr, host, lens, np.stack(prevs), G)
    assert np.array_equal(got, oracle.topk_batched(host, K, row_lens=lens)), st.tolist()
    assert all(int(s[7]) == G for s in st)


@pytest.mark.parametrize("G", [2, 8])
@pytest.mark.parametrize("gk", ["random", "adversarial", "none", "all_minus1"])
def test_cluster_guess_kinds(gvr, G, gk):
    n = 120_000
    p, c = synth.decode_pair(n, 0.9, seed=610)
    row = c.numpy()
    host, lens = _pack([row])
    g = synth.guess(gk, row, K, 611)
    got, st = _run_cluster(gvr, host, lens, None if g is None else g[None, :], G)
    assert np.array_equal(got, oracle.topk_batched(host, K, row_lens=lens)), st.tolist()


@pytest.mark.parametrize("kind", ["ties90", "few_distinct", "signed_zero_mix", "with_inf", "normal"])
def test_cluster_distributions(gvr, kind):
    rows = [synth.dist_row(kind, n, seed=620 + i) for i, n in enumerate([70_000, 33_000, 131_072])]
    host, lens = _pack(rows)
    prev = np.stack([synth.guess("random", r, K, 9) for r in rows])
    for G in (4, 8):
        got, st = _run_cluster(gvr, host, lens, prev, G)
        assert np.array_equal(got, oracle.topk_batched(host, K, row_lens=lens)), (G, st.tolist())


def test_cluster_ragged_and_trivial_rows(gvr):
    rows = [synth.dist_row("normal", n, seed=630 + i) for i, n in enumerate([0, 5, 2048, 2049, 40_000, 99_999])]
    host, lens = _pack(rows, stride=100_003)
    got, st = _run_cluster(gvr, host, lens, None, 8)
    assert np.array_equal(got, oracle.topk_batched(host, K, row_lens=lens)), st.tolist()


def test_cluster_chosen_automatically_at_batch_1(gvr):
    import torch
    n = 131_072
    p, c = synth.decode_pair(n, 0.9, seed=640)
    host, lens = _pack([c.numpy()])
    prev = oracle.topk(p.numpy(), K)[None, :]
    dev = torch.device("cuda:0")
    idx, _, st = gvr.topk_ex(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                             prev=torch.from_numpy(prev).to(dev))
    torch.cuda.synchronize()
    assert np.array_equal(idx.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))
    assert int(st.cpu().numpy()[0, 7]) == 8


@pytest.mark.parametrize("gk", ["prev", "random", "adversarial"])
def test_guess_stride_never_changes_result(gvr, gk):
    """Phase-1 statistics over every guess_stride-th guessed position (R29) change only the
    collect threshold, never the output: strides 1 (the paper's all positions), 2, 4."""
    import torch
    dev = torch.device("cuda:0")
    rows, prevs = [], []
    for i in range(5):
        p, c = synth.decode_pair(90_000, 0.9 if i % 2 else 0.0, seed=700 + i)
        rows.append(c.numpy())
        prevs.append(synth.guess(gk, rows[-1], K, 701 + i, prev_topk=oracle.topk(p.numpy(), K)))
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, K, row_lens=lens)
    s = torch.from_numpy(host).to(dev)
    l = torch.from_numpy(lens).to(dev)
    pv = torch.from_numpy(np.stack(prevs).astype(np.int32)).to(dev)
    for stride in (1, 2, 4):
        idx, _, _ = gvr.topk_ex(s, K, row_lens=l, prev=pv, options=gvr.GvrOptions(float("nan"), 0, 0, stride))
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), ref), stride


@pytest.mark.parametrize("n", [8192, 20_000, 100_000, 262_144])
def test_guess_overshoot_takes_a_second_pass(gvr, n):
    """f(T_c) < K (a Phase-2 window aimed below the K-th value, window_z = -8) -> the row
    is streamed once more at pmin of a complete guess / -inf (R30): exact result, two
    HBM passes; the default window never needs it on these rows."""
    import torch
    dev = torch.device("cuda:0")
    rows = [synth.dist_row(kind, n, seed=800 + i) for i, kind in enumerate(["normal", "lognormal", "uniform"])]
    p, c = synth.decode_pair(n, 0.9, seed=810)
    rows.append(c.numpy())
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, K, row_lens=lens)
    perfect = np.stack([oracle.topk(r, K) for r in rows]).astype(np.int32)  # the current Top-K itself
    s = torch.from_numpy(host).to(dev)
    l = torch.from_numpy(lens).to(dev)
    for z, stride in ((float("nan"), 1), (-8.0, 1), (-8.0, 4)):
        idx, _, st = gvr.topk_ex(s, K, row_lens=l, prev=torch.from_numpy(perfect).to(dev),
                                 options=gvr.GvrOptions(z, 0, 0, stride))
        torch.cuda.synchronize()
        st = st.cpu().numpy()
        assert np.array_equal(idx.cpu().numpy(), ref), (z, stride, st.tolist())
        if z < 0:
            # two passes, converged (at N = 8192 the sample is half the row, so the window
            # may still admit pmin of the perfect guess, which is exactly the K-th value)
            assert (st[:, 4] <= 2).all() and (st[:, 3] == 1).all(), st.tolist()
            if n > 8192:
                assert (st[:, 4] == 2).all(), st.tolist()
        else:
            assert (st[:, 4] == 1).all(), st.tolist()


@pytest.mark.parametrize("path", [0, 1])
def test_split_path_ragged_trivial_and_mixed_guesses(gvr, path):
    """More than one wave of rows (guess kernel, then the filter + refine kernels (path 0)
    or the row streaming kernel (path 1)): ragged lengths including empty and len <= k
    rows, every guess kind, value distributions; exact against the oracle."""
    import torch
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(11)
    R = 340  # > 2 x 148 resident CTAs: the split path
    lens = rng.integers(0, 40_000, size=R).astype(np.int32)
    lens[:6] = [0, 1, 2047, 2048, 2049, 40_000]
    S = int(lens.max())
    host = np.zeros((R, S), np.float32)
    kinds = synth.DISTRIBUTIONS
    prev = np.full((R, K), -1, np.int32)
    for r in range(R):
        n = int(lens[r])
        if n == 0:
            continue
        row = synth.dist_row(kinds[r % len(kinds)], n, seed=900 + r)
        host[r, :n] = row
        g = synth.guess(synth.GUESS_KINDS[r % 6], row, K, 901 + r, prev_topk=oracle.topk(row, K))
        if g is not None:
            prev[r] = g
    ref = oracle.topk_batched(host, K, row_lens=lens)
    out = gvr.topk(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                   prev=torch.from_numpy(prev).to(dev), options=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    bad = np.argwhere((got != ref).any(axis=1))[:, 0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5].tolist()} lens {lens[bad[:5]].tolist()}"


def _filter_batch(gvr, host, lens, prev, k=K, path=0):
    import torch
    dev = torch.device("cuda:0")
    p = None if prev is None else torch.from_numpy(np.ascontiguousarray(prev, np.int32)).to(dev)
    idx, val, st = gvr.topk_ex(torch.from_numpy(host).to(dev), k, row_lens=torch.from_numpy(lens).to(dev), prev=p,
                               options=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
    torch.cuda.synchronize()
    return idx.cpu().numpy(), val.cpu().numpy(), st.cpu().numpy()


def _assert_rows(got, ref, lens, st=None):
    bad = np.argwhere((got != ref).any(axis=1))[:, 0]
    assert bad.size == 0, (f"{bad.size} rows differ, first {bad[:5].tolist()} lens {lens[bad[:5]].tolist()}"
                           + ("" if st is None else f" stats {st[bad[:3]].tolist()}"))


@pytest.mark.parametrize("stride_pad", [0, 1, 2, 3, 5])
def test_filter_path_misaligned_rows(gvr, stride_pad):
    """Filter path with row strides that are not a multiple of 4 floats: every row has its
    own unaligned head and tail scalars, handled in the rounds holding its first and last
    tiles; some rows span several filter CTAs."""
    R, n = 320, 30_000 + stride_pad
    rows = [synth.dist_row(synth.DISTRIBUTIONS[r % len(synth.DISTRIBUTIONS)], n - (r % 4), seed=1000 + r)
            for r in range(R)]
    host, lens = _pack(rows, stride=n)
    prev = np.full((R, K), -1, np.int32)
    for r in range(R):
        g = synth.guess(synth.GUESS_KINDS[r % len(synth.GUESS_KINDS)], rows[r], K, 1001 + r,
                        prev_topk=oracle.topk(rows[r], K))
        if g is not None:
            prev[r] = g
    ref = oracle.topk_batched(host, K, row_lens=lens)
    got, val, st = _filter_batch(gvr, host, lens, prev)
    _assert_rows(got, ref, lens, st)
    for r in range(0, R, 17):
        m = min(K, lens[r])
        assert np.array_equal(val[r, :m].view(np.uint32), host[r, ref[r, :m]].view(np.uint32))


@pytest.mark.parametrize("k", [1, 7, 100, 1000, 2047])
def test_filter_path_small_k(gvr, k):
    R, n = 310, 9_000
    rows = [synth.dist_row("normal", n, seed=1100 + r) for r in range(R)]
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, k, row_lens=lens)
    prev = np.stack([oracle.topk(synth.dist_row("normal", n, seed=1100 + r + 1), k) for r in range(R)])
    got, _, st = _filter_batch(gvr, host, lens, prev, k=k)
    _assert_rows(got, ref, lens, st)


def test_filter_path_poor_guesses_and_long_lists(gvr):
    """Rows whose guess says nothing (rho = 0, layers 0-1 of DSV3.2): the guess kernel takes
    the threshold from a row sample; rows whose list exceeds the shared-memory buffer are
    cut by the count search; rows with massive ties or overflowing lists are streamed
    again by the refine kernel.  Exact in every case, with stats consistent."""
    R, n = 300, 100_000
    rows, prevs = [], []
    for r in range(R):
        kind = r % 5
        if kind == 0:
            p, c = synth.decode_pair(n, 0.0, seed=1200 + r)
            rows.append(c.numpy())
            prevs.append(oracle.topk(p.numpy(), K))
        elif kind == 1:
            p, c = synth.decode_pair(n, 0.9, seed=1200 + r)
            rows.append(c.numpy())
            prevs.append(oracle.topk(p.numpy(), K))
        elif kind == 2:
            row = synth.dist_row(("few_distinct", "all_equal", "ties90")[(r // 5) % 3], n, seed=1200 + r)
            rows.append(row)
            prevs.append(synth.guess("random", row, K, 1201 + r))
        elif kind == 3:
            row = synth.dist_row("normal", n, seed=1200 + r)
            rows.append(row)
            prevs.append(synth.guess("adversarial", row, K, 1201 + r, prev_topk=oracle.topk(row, K)))
        else:
            row = synth.dist_row("normal", n, seed=1200 + r)
            rows.append(row)
            prevs.append(None)
    prev = np.stack([p if p is not None else np.full(K, -1, np.int32) for p in prevs])
    host, lens = _pack(rows)
    ref = oracle.topk_batched(host, K, row_lens=lens)
    got, _, st = _filter_batch(gvr, host, lens, prev)
    _assert_rows(got, ref, lens, st)
    assert (st[:, 4] >= 1).all()  # global passes
    good = st[1::5]
    assert (good[:, 4] == 1).all() and (good[:, 3] == 1).all(), good[:5].tolist()  # one pass, converged


def test_filter_path_cuda_graph(gvr):
    """The three-kernel filter path (guess, filter, refine) and its scratch capture into a
    CUDA graph; replays on new inputs written into the same buffers are exact."""
    import torch
    dev = torch.device("cuda:0")
    host_a, lens, prev_a = _decode_rows(300, n=12_000, seed=1300)
    host_b, _, prev_b = _decode_rows(300, n=12_000, seed=1400)
    s = torch.from_numpy(host_a).to(dev)
    l = torch.from_numpy(lens).to(dev)
    p = torch.from_numpy(prev_a).to(dev)
    out = torch.empty((300, K), dtype=torch.int32, device=dev)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        gvr.topk(s, K, row_lens=l, prev=p, out=out)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gvr.topk(s, K, row_lens=l, prev=p, out=out)
    for host, prev in ((host_a, prev_a), (host_b, prev_b)):
        s.copy_(torch.from_numpy(host))
        p.copy_(torch.from_numpy(prev))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens))


def test_filter_and_row_paths_agree_on_cfg4(gvr):
    """BASELINE.json configs[3] shape (MTP: 4 draft rows per request, N + j keys) at 16
    requests x 8 layers: both batch paths equal the oracle."""
    import torch
    from bench import make_decode_batch
    dev = torch.device("cuda:0")
    batch = make_decode_batch(16, 8, 100_000, dev, seed=synth.BASE_SEED + 7, draft=4)
    torch.cuda.synchronize()
    host = batch["scores"].cpu().numpy()
    lens = batch["row_lens"].cpu().numpy()
    ref = oracle.topk_batched(host, K, row_lens=lens)
    for path in (0, 1):
        out = gvr.topk(batch["scores"], K, row_lens=batch["row_lens"], prev=batch["prev"],
                       options=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
        torch.cuda.synchronize()
        _assert_rows(out.cpu().numpy(), ref, lens)


def test_filter_path_alternating_batch_sizes_and_paths(gvr):
    """The per-stream scratch (ready queue, control words, candidate regions) is reused
    across calls of different batch sizes, row lengths and batch paths: every call is
    exact.  (Its zero words live at fixed offsets sized by the lease's row capacity.)"""
    import torch
    dev = torch.device("cuda:0")
    jobs = [(320, 12_000, 0), (488, 20_000, 0), (300, 9_000, 0), (330, 16_000, 1), (420, 7_000, 0),
            (300, 12_000, 0)]
    for i, (R, n, path) in enumerate(jobs):
        rng = np.random.default_rng(1500 + i)
        host = rng.standard_normal((R, n)).astype(np.float32)
        lens = rng.integers(n // 2, n + 1, size=R).astype(np.int32)
        # a correlated previous step: the Top-K of a noisy copy of each row
        prev = oracle.topk_batched(host + 0.3 * rng.standard_normal((R, n)).astype(np.float32), K, row_lens=lens)
        out = gvr.topk(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                       prev=torch.from_numpy(prev).to(dev), options=gvr.GvrOptions(float("nan"), 0, 0, 0, path))
        torch.cuda.synchronize()
        _assert_rows(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens), lens)


@pytest.mark.parametrize("R", [400, 1100])
def test_refine_lists_longer_than_the_held_registers(gvr, R):
    """Both refine geometries (R <= 1024: 512 threads x 8 held entries; R > 1024: 256 x 16)
    hold 4,096 list entries per row in registers and re-read the rest from L2 on every
    pass.  A wide Phase-2 window (window_z = 30) lowers T_c until most lists exceed 4,096
    entries: exact; the rows refined from their lists had more than 4,096 candidates."""
    import torch
    dev = torch.device("cuda:0")
    n = 30_000
    rng = np.random.default_rng(2800 + R)
    host = rng.standard_normal((R, n)).astype(np.float32)
    lens = np.full(R, n, np.int32)
    out, _, st = gvr.topk_ex(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev),
                             options=gvr.GvrOptions(30.0, 0, 0, 0, 0))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    _assert_rows(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens), lens, st)
    # most rows were refined from lists longer than the held capacity, in one HBM pass (at
    # R = 1100 some CTA regions overflow: those rows are streamed again by the fixup — exact)
    long_rows = st[:, 2] > 4096
    assert long_rows.mean() > 0.5, np.percentile(st[:, 2], [0, 50, 100])
    assert (st[long_rows, 4] == 1).all()


def test_refine_zooms_into_a_crowded_lowest_bin(gvr):
    """Rows whose candidate list is a dense cluster of negative scores plus a few far
    positive outliers: in linear key bins over [T_c, max] nearly every entry falls into the
    lowest bin, which is also the K-th bin.  The refine zooms into that bin from above
    (the outliers saturate into bin 0) instead of ranking thousands of entries in one
    bin: exact, refined from the lists, three histogram levels."""
    import torch
    dev = torch.device("cuda:0")
    R, n = 320, 30_000
    rng = np.random.default_rng(2900)
    host = (-1.0 + 1e-3 * rng.standard_normal((R, n))).astype(np.float32)
    for r in range(R):
        host[r, rng.choice(n, 12, replace=False)] = (100.0 + 50 * rng.random(12)).astype(np.float32)
    lens = np.full(R, n, np.int32)
    out, _, st = gvr.topk_ex(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    _assert_rows(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens), lens, st)
    assert (st[:, 5] >= 1).mean() > 0.9, np.bincount(st[:, 5])  # narrowed / zoomed
    assert (st[:, 1] == 0).all()  # no row needed the fixup kernel (its snap iterations)


def test_threshold_handoff_never_reads_a_stale_generation(gvr):
    """The filter kernel takes each row's T_c from a generation-tagged word (BatchQueue::tcw)
    instead of waiting for the guess grid.  Rows of a shrinking then growing batch on one
    stream reuse words written by earlier calls with other thresholds: every call must be
    exact (a stale word would hand a row another call's T_c — too high drops rows of the
    Top-K from the list, too low overflows it)."""
    import torch
    dev = torch.device("cuda:0")
    for i, (R, scale) in enumerate([(480, 1.0), (310, 50.0), (480, -3.0), (300, 0.01), (480, 1.0)]):
        rng = np.random.default_rng(2600 + i)
        n = 9_000 + 1_000 * i
        host = (scale * rng.standard_normal((R, n))).astype(np.float32)
        lens = np.full(R, n, np.int32)
        out = gvr.topk(torch.from_numpy(host).to(dev), K, row_lens=torch.from_numpy(lens).to(dev))
        torch.cuda.synchronize()
        _assert_rows(out.cpu().numpy(), oracle.topk_batched(host, K, row_lens=lens), lens)


def test_cta_timeline_diagnostic(gvr):
    """gvr_cta_timeline records, per filter CTA, entry <= first-threshold <= exit and an SM
    id, and per guess CTA entry <= loads arrived <= Phase 1 done <= exit."""
    import torch
    dev = torch.device("cuda:0")
    R, n = 400, 20_000
    rng = np.random.default_rng(2700)
    host = rng.standard_normal((R, n)).astype(np.float32)
    scores = torch.from_numpy(host).to(dev)
    gvr.topk(scores, K)
    torch.cuda.synchronize()
    gvr.cta_timeline(True)
    out = gvr.topk(scores, K)
    ft = gvr.cta_timeline(False, "filter")
    gt = gvr.cta_timeline(False, "guess")[:R]
    _assert_rows(out.cpu().numpy(), oracle.topk_batched(host, K), np.full(R, n, np.int32))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ft = ft[:3 * sms]
    ran = ft[:, 2] > 0
    assert ran.sum() > 0
    f = ft[ran]
    assert np.all(f[:, 0] <= f[:, 1]) and np.all(f[:, 1] <= f[:, 2])
    assert np.all((f[:, 3] >= 0) & (f[:, 3] < sms))
    assert np.all(gt[:, 0] <= gt[:, 2]) and np.all(gt[:, 2] <= gt[:, 3]) and np.all(gt[:, 3] <= gt[:, 1])
    # every filter CTA starts its stream only after some guess CTA finished
    assert f[:, 1].min() >= gt[:, 1].min()


# ------------------------------------------------------------------ scratch lease
def test_graph_captured_on_warm_stream_survives_eager_growth(gvr):
    """Warm up and capture on the SAME stream (the cache already holds a big-enough slot),
    then grow that stream's slot with a larger eager call, then replay: the graph owns its
    own scratch, so the replay is exact."""
    import torch
    dev = torch.device("cuda:0")
    host_a, lens, prev_a = _decode_rows(300, n=12_000, seed=1600)
    host_big, lens_big, prev_big = _decode_rows(600, n=12_000, seed=1601)
    s = torch.from_numpy(host_a).to(dev)
    l = torch.from_numpy(lens).to(dev)
    p = torch.from_numpy(prev_a).to(dev)
    out = torch.empty((300, K), dtype=torch.int32, device=dev)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        gvr.topk(s, K, row_lens=l, prev=p, out=out)  # sizes the stream's slot
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            gvr.topk(s, K, row_lens=l, prev=p, out=out)
        big = gvr.topk(torch.from_numpy(host_big).to(dev), K, row_lens=torch.from_numpy(lens_big).to(dev),
                       prev=torch.from_numpy(prev_big).to(dev))  # grows (and frees) the slot
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.topk_batched(host_a, K, row_lens=lens))
    assert np.array_equal(big.cpu().numpy(), oracle.topk_batched(host_big, K, row_lens=lens_big))


def test_per_thread_default_streams_from_two_host_threads(gvr):
    """Two host threads each call GVR on their own per-thread default stream (one handle
    value, two streams): each keeps its own scratch lease."""
    import threading

    import torch
    dev = torch.device("cuda:0")
    jobs = [_decode_rows(300, n=9_000, seed=1700 + i) for i in range(2)]
    results, errors = [None, None], []

    def work(i):
        try:
            torch.cuda.set_device(dev)
            host, lens, prev = jobs[i]
            s = torch.from_numpy(host).to(dev)
            l = torch.from_numpy(lens).to(dev)
            p = torch.from_numpy(prev).to(dev)
            ptd = torch.cuda.ExternalStream(2)  # cudaStreamPerThread
            outs = [gvr.topk(s, K, row_lens=l, prev=p, stream=ptd) for _ in range(4)]
            torch.cuda.synchronize()
            results[i] = [o.cpu().numpy() for o in outs]
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (host, lens, _), res in zip(jobs, results):
        ref = oracle.topk_batched(host, K, row_lens=lens)
        for o in res:
            assert np.array_equal(o, ref)
