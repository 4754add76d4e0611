"""The multi-rank GPU executor (csrc/tile.cpp over csrc/dist.cpp) on ONE B200:
P x Q ranks simulated in one process (mp_dist_create_sim), each rank with its
own context and streams, driven from its own host thread; the broadcasts are
event-ordered device copies between the ranks' buffers (no kernel waits on
another rank's).  Everything else — the row/column schedule, the per-rank
work lists, the head/tail TRSM split, the panel conversions on the receiving
ranks, the failing-pivot reduction, the distributed logdet and NLL forward
solve — is the code an NCCL run executes.  The gathered factor must equal the
single-GPU factor bit for bit (every tile is computed by the same kernels
from the same operands)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(fns):
    errs = [None] * len(fns)
    out = [None] * len(fns)

    def go(r):
        try:
            out[r] = fns[r]()
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=go, args=(r,)) for r in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "simulated ranks hung"
    for e in errs:
        if e is not None:
            raise e
    return out


def _band(nt, b64, b32):
    i, j = np.indices((nt, nt))
    d = abs(i - j)
    return np.where(d < b64, 2, np.where(d < b32, 1, 0)).astype(np.int32)


@pytest.mark.parametrize("P,Q,b64,b32", [(1, 2, 1, 2), (2, 1, 1, 3), (2, 2, 1, 3), (2, 2, 2, 4), (1, 3, 1, 2)])
def test_dist_executor_simulated_ranks_bitwise(P, Q, b64, b32):
    import paper_2406_02701_b200 as mp

    n, nb, side = 4096, 256, 64
    nt = n // nb
    g = _band(nt, b64, b32)
    ctx0 = mp.Context(0)
    a = mp.MPCRTile(n, n, nb, nb, None, g, ctx0)
    a.fill_matern(side, 0.5, 0.03, 1.0)
    mp.tile_chol(a)
    La, lda = a.to_numpy(), a.logdet()
    world = P * Q
    ctxs = [mp.Context(0) for _ in range(world)]
    grids = mp.ProcessGrid.simulated(ctxs, P, Q)
    tiles = [mp.MPCRTile(n, n, nb, nb, None, g, ctxs[r], grid=grids[r]) for r in range(world)]
    for r, t in enumerate(tiles):
        t.fill_matern(side, 0.5, 0.03, 1.0)
        ctxs[r].synchronize()
    for _ in range(2):  # twice: the executor's cached plans / events are reused
        for r in range(world):
            t2 = tiles[r]
            t2.fill_matern(side, 0.5, 0.03, 1.0)
            ctxs[r].synchronize()
        _run_ranks([lambda t=t: mp.tile_chol(t) for t in tiles])
        L = sum(t.to_numpy() for t in tiles)
        assert np.array_equal(L, La)
    lds = _run_ranks([lambda t=t: t.logdet() for t in tiles])
    assert all(abs(x - lda) <= 1e-12 * abs(lda) for x in lds), (lds, lda)
    for r in range(world):
        for i in range(nt):
            for j in range(i + 1):
                assert tiles[r].owns(i, j) == (mp.dist_owner(i, j, P, Q) == r)


def test_dist_simulated_nll_and_failing_pivot():
    """The distributed NLL (forward solve segment by segment over the ranks)
    equals the single-GPU one; a non-SPD matrix reports the same global
    failing column on every rank."""
    import paper_2406_02701_b200 as mp

    n, nb, P, Q = 2048, 256, 2, 2
    nt = n // nb
    g = _band(nt, 1, 3)
    x = np.random.default_rng(1).random(n)
    y = np.random.default_rng(2).random(n)
    z = mp.rng_normal(4, n)
    ctx0 = mp.Context(0)
    a = mp.MPCRTile(n, n, nb, nb, None, g, ctx0)
    a.fill_matern_points(x, y, 0.5, 0.1, 1.0, 0.0)
    want = mp.gaussian_nll(z, a, jitter=1e-6, max_jitter=1e-3)
    ctxs = [mp.Context(0) for _ in range(P * Q)]
    grids = mp.ProcessGrid.simulated(ctxs, P, Q)
    tiles = [mp.MPCRTile(n, n, nb, nb, None, g, ctxs[r], grid=grids[r]) for r in range(P * Q)]
    for t in tiles:
        t.fill_matern_points(x, y, 0.5, 0.1, 1.0, 0.0)
    got = _run_ranks([lambda t=t: mp.gaussian_nll(z, t, jitter=1e-6, max_jitter=1e-3) for t in tiles])
    for r in got:
        assert r["jitter"] == want["jitter"]
        assert abs(r["logdet"] - want["logdet"]) <= 1e-10 * abs(want["logdet"])
        assert abs(r["nll"] - want["nll"]) <= 1e-10 * abs(want["nll"])
    # not positive definite at global column 3 * nb + 17: every rank reports it
    M = np.eye(n)
    M[3 * nb + 17, 3 * nb + 17] = -1.0
    bad = [mp.MPCRTile(n, n, nb, nb, M, np.full((nt, nt), 2, np.int32), ctxs[r], grid=grids[r]) for r in range(P * Q)]

    def chol_info(t):
        try:
            mp.tile_chol(t)
        except mp.MPError as e:
            return e.kind, e.info
        return None

    res = _run_ranks([lambda t=t: chol_info(t) for t in bad])
    assert res == [("NotPositiveDefinite", 3 * nb + 17)] * (P * Q), res
