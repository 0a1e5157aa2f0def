"""CPU pins of the seeded synthetic input generator (synth/)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def test_yarn_inv_freq_closed_forms():
    f = synth.yarn_inv_freq().double().numpy()
    assert f.shape == (32,)
    # i = 0 lies below the ramp (lo = 10): unscaled theta_0 = base^0 = 1
    assert f[0] == pytest.approx(1.0)
    # i = 31 lies above the ramp (hi = 23): theta_31 / 40 = 1e4^(-62/64) / 40
    assert f[31] == pytest.approx(1e4 ** (-62 / 64) / 40, rel=1e-6)
    # inside the ramp the value is between the interpolated and extrapolated frequencies
    th = 1e4 ** (-np.arange(0, 64, 2) / 64)
    assert np.all(f <= th * (1 + 1e-6)) and np.all(f >= th / 40 * (1 - 1e-6))
    assert np.all(np.diff(f) < 0)


def test_g_delta_closed_forms():
    g = synth.g_delta(100)
    assert g[0] == pytest.approx(64.0)  # 2 * 32 * cos(0)
    assert np.all(g <= 64.0 + 1e-9)


def test_static_prior_valid_positions():
    n = 20_000
    p = synth.static_prior(n, 2048)
    assert p.dtype == np.int32 and p.shape == (2048,)
    assert len(set(p.tolist())) == 2048
    assert p.min() >= 0 and p.max() == n - 1  # Delta = 0 is the global maximum of g
    short = synth.static_prior(100, 2048)
    assert (short[:100] >= 0).all() and (short[100:] == -1).all()
    p0 = synth.static_prior(n, 2048, query_pos=0)
    assert 0 in set(p0.tolist())  # Delta = 0 is position 0 when the query sits there
    assert sorted(p0.tolist()) == sorted((n - 1 - p).tolist())  # mirror image


def test_static_prior_matches_appendix_e_rows():
    """App.-E rows (query at position 0) are dominated by g(Delta):
    the prior built for query_pos=0 overlaps the exact Top-K far above chance (K/N),
    the mirrored one (query at the end) does not."""
    import oracle
    n, k = 16384, 2048
    row = synth.appendix_e_row(n, seed=5).numpy()
    top = set(oracle.topk(row, k).tolist())
    a0 = len(top & set(synth.static_prior(n, k, query_pos=0).tolist())) / k
    a_end = len(top & set(synth.static_prior(n, k).tolist())) / k
    assert a0 > 0.5 > a_end


def test_rope_is_a_rotation_and_relative():
    g = torch.Generator().manual_seed(0)
    inv = synth.yarn_inv_freq()
    q = torch.randn(64, generator=g, dtype=torch.float32)
    k = torch.randn(64, generator=g, dtype=torch.float32)
    for m in (0, 7, 1000):
        qr = synth.rope_rotate(q[None], torch.tensor([m]), inv)[0]
        assert torch.linalg.norm(qr).item() == pytest.approx(torch.linalg.norm(q).item(), rel=1e-5)
    # <R(a) q, R(b) k> depends only on a - b
    def dot(a, b):
        qa = synth.rope_rotate(q[None].double(), torch.tensor([a]), inv.double())[0]
        kb = synth.rope_rotate(k[None].double(), torch.tensor([b]), inv.double())[0]
        return float(qa @ kb)
    assert dot(50, 20) == pytest.approx(dot(130, 100), rel=1e-9, abs=1e-9)


def test_indexer_scores_match_eq1_definition():
    n = 300
    lay = synth.IndexerLayer(n, 0.9, seed=5)
    row = lay.scores(n).double()
    q = lay.q.clone().double()
    q[:, :64] = synth.rope_rotate(q[:, :64], torch.full((64,), n - 1), lay.inv_freq.double())
    ref = (lay.w.double()[:, None] * torch.relu(q @ lay.keys[:n].double().T)).sum(0)
    assert torch.allclose(row, ref, rtol=1e-4, atol=1e-4)


def test_generator_is_deterministic():
    a = synth.decode_pair(2000, 0.9, seed=3)
    b = synth.decode_pair(2000, 0.9, seed=3)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    c = synth.decode_pair(2000, 0.9, seed=4)
    assert not torch.equal(a[1], c[1])
    assert np.array_equal(synth.dist_row("ties90", 1000, 2), synth.dist_row("ties90", 1000, 2))


def test_temporal_hit_ratio_calibration():
    """AR(1) rho controls the consecutive-step Top-K overlap alpha (PAPER.md:275-277,
    372-377): rho = 0.9 gives alpha in the L20-60 band region, rho = 0 near K/N."""
    n, K = 16384, 2048

    def alpha(rho, seed):
        p, c = synth.decode_pair(n, rho, seed)
        a = set(oracle.topk(p.numpy(), K).tolist())
        b = set(oracle.topk(c.numpy(), K).tolist())
        return len(a & b) / K

    hi = np.mean([alpha(0.9, s) for s in range(3)])
    lo = np.mean([alpha(0.0, s) for s in range(3)])
    assert 0.35 <= hi <= 0.8
    assert lo <= 0.3
    assert hi > lo + 0.2


@pytest.mark.parametrize("kind", synth.DISTRIBUTIONS)
def test_dist_rows(kind):
    r = synth.dist_row(kind, 777, seed=1)
    assert r.dtype == np.float32 and r.shape == (777,)


@pytest.mark.parametrize("kind", synth.GUESS_KINDS)
def test_guess_kinds(kind):
    row = synth.dist_row("normal", 5000, 1)
    g = synth.guess(kind, row, 2048, 1, prev_topk=np.arange(2048, dtype=np.int32))
    if kind == "none":
        assert g is None
    else:
        assert g.dtype == np.int32 and g.shape == (2048,)


def test_layer_rho_bands():
    assert synth.layer_rho(0, 1) == 0.0 and synth.layer_rho(1, 1) == 0.0
    for l in range(2, 61):
        assert 0.88 <= synth.layer_rho(l, 1) <= 0.93
