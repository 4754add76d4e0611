"""GPU parity: the Gaussian log-likelihood pipeline (config 5): Matern
covariance generated on the device -> (jittered) tiled Cholesky -> tiled
forward solve -> logdet / quadratic form -> nll, against the reference's
gaussian_nll (workloads.cpp:74-87) and the composed MPCRTile oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def grid(n):
    side = int(np.ceil(np.sqrt(n)))
    p = np.arange(n)
    return (p % side) / (side - 1), (p // side) / (side - 1), side


def test_nll_identity(ctx):
    """nll(I, z=0) = n/2 log 2 pi (test_stats.cpp:152-160)."""
    import paper_2406_02701_b200 as mp

    n = 256
    t = mp.MPCRTile(n, n, 64, 64, np.eye(n), np.full((4, 4), 2), ctx)
    r = mp.gaussian_nll(np.zeros(n), t, jitter=0.0)
    assert abs(r["nll"] - 0.5 * n * np.log(2 * np.pi)) < 1e-12
    assert r["logdet"] == 0.0 and r["quad"] == 0.0


@pytest.mark.parametrize("prec", [1, 2])
def test_nll_matches_reference_uniform_precision(ctx, ref, prec):
    """All tiles at one precision == the reference's gaussian_nll at that
    precision (its jitter policy included)."""
    import paper_2406_02701_b200 as mp

    n, nb = 400, 100
    x, y, side = grid(n)
    cov = ref.grid_matern(side, n, 0.5, 0.1, 1.0, 2)
    z = ref.sample_gp(cov, 4)
    want = ref.gaussian_nll(prec, z, cov)
    t = mp.MPCRTile(n, n, nb, nb, None, np.full((4, 4), prec), ctx)
    t.fill_matern(side, 0.5, 0.1, 1.0)
    got = mp.gaussian_nll(z, t, jitter=1e-6 if prec != 2 else 0.0)
    tol = 1e-10 if prec == 2 else 1e-3
    assert abs(got["nll"] - want) <= tol * abs(want), (got, want)


def test_nll_mixed_vs_composed_oracle(ctx, ref):
    """Mixed map: nll from the GPU factor vs nll from the composed oracle's
    factor (same map), solved in FP64 on the host."""
    import paper_2406_02701_b200 as mp

    n, nb = 1024, 128
    x, y, side = grid(n)
    cov = ref.grid_matern(side, n, 0.5, 0.03, 1.0, 2)
    z = ref.sample_gp(cov, 4)
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    t.fill_matern_points(x, y, 0.5, 0.03, 1.0, 0.0)
    got = mp.gaussian_nll(z, t, jitter=0.0)
    L = ref.tile_chol(n, nb, g, cov)
    import scipy.linalg as sl

    w = sl.solve_triangular(L, z, lower=True)
    want = 0.5 * w @ w + np.log(np.diag(L)).sum() + 0.5 * n * np.log(2 * np.pi)
    exact = ref.gaussian_nll(2, z, cov)
    assert abs(got["nll"] - want) <= max(4 * abs(want - exact), 1e-9 * abs(exact)), (got, want, exact)


def test_nll_jitter_escalation(ctx):
    """A matrix that needs jitter: the first attempts fail, escalation x10
    succeeds (workloads.cpp:63-67); without jitter it reports NotPD."""
    import paper_2406_02701_b200 as mp

    n = 128
    v = np.ones(n) / np.sqrt(n)
    M = np.eye(n) - np.outer(v, v) * (1 - 1e-9)  # nearly singular PSD
    M[0, 0] -= 5e-3  # lambda_min ~ -5e-3 / n ~ -3.9e-5: needs jitter 1e-4
    t = mp.MPCRTile(n, n, 32, 32, M, np.full((4, 4), 2), ctx)
    r = mp.gaussian_nll(np.ones(n), t, jitter=1e-6, max_jitter=1e-3)
    assert r["jitter"] >= 0.99e-4  # 1e-6 x 10 x 10
    t2 = mp.MPCRTile(n, n, 32, 32, M, np.full((4, 4), 2), ctx)
    with pytest.raises(mp.MPError) as e:
        mp.gaussian_nll(np.ones(n), t2, jitter=0.0)
    assert e.value.kind == "NotPositiveDefinite"


def test_matern_mle_matches_reference(ctx, ref):
    """matern_mle (workloads.cpp:89-110): the same Nelder-Mead path as the
    reference (identical iteration count) with every likelihood on the GPU;
    all-FP64 tiles against the reference's Double run (no jitter)."""
    import paper_2406_02701_b200 as mp

    side, n, nb = 20, 400, 100
    x, y, _ = grid(n)
    cov = ref.grid_matern(side, n, 0.5, 0.1, 1.0, 2)
    z = ref.sample_gp(cov, 4)
    want = ref.matern_mle(2, side, z, np.log(0.05), np.log(0.5), 200, 1e-4)
    t = mp.MPCRTile(n, n, nb, nb, None, np.full((4, 4), 2), ctx)
    got = mp.matern_mle(t, x, y, z, np.log(0.05), np.log(0.5), max_iter=200, tol=1e-4, jitter=0.0)
    assert got["converged"]
    assert got["iterations"] == want["iterations"], (got, want)
    assert abs(got["range"] - want["range"]) <= 1e-8 * want["range"], (got, want)
    assert abs(got["sigma2"] - want["sigma2"]) <= 1e-8 * want["sigma2"], (got, want)
    assert abs(got["nll"] - want["nll"]) <= 1e-10 * abs(want["nll"]), (got, want)


def test_matern_mle_mixed_precision_close(ctx, ref):
    """A mixed FP64/FP32/FP16 tile map reaches the FP64 optimum to the
    precision the FP16 tiles allow."""
    import paper_2406_02701_b200 as mp

    side, n, nb = 32, 1024, 128
    x, y, _ = grid(n)
    z = ref.sample_gp(ref.grid_matern(side, n, 0.5, 0.05, 1.0, 2), 4)
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    t64 = mp.MPCRTile(n, n, nb, nb, None, np.full((nt, nt), 2), ctx)
    tmx = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    a = mp.matern_mle(t64, x, y, z, np.log(0.03), np.log(0.7), jitter=0.0)
    b = mp.matern_mle(tmx, x, y, z, np.log(0.03), np.log(0.7), jitter=1e-6)
    assert a["converged"] and b["converged"]
    assert abs(b["range"] - a["range"]) <= 2e-2 * a["range"], (a, b)
    assert abs(b["sigma2"] - a["sigma2"]) <= 2e-2 * a["sigma2"], (a, b)
