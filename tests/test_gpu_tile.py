"""GPU parity: MPCRTile vs the composed reference oracle
(oracle/ref_shim.cpp: ref_tile_chol / ref_tile_gemm / ref_tile_trsm) and the
paper's printed known answers."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, S, D = 0, 1, 2


def paper_M():
    xs = np.array([(x, y) for y in (0.0, 1.0) for x in (0.0, 1.0)])
    d = np.sqrt(((xs[:, None] - xs[None]) ** 2).sum(-1))
    return np.exp(-d)


def test_paper_chol_4x4(ctx, ref):
    """PAPER.md:585-588 (diag double, off-diag single, 2x2 tiles)."""
    import paper_2406_02701_b200 as mp

    M = paper_M()
    prec = [["double", "single"], ["single", "double"]]
    t = mp.MPCRTile(4, 4, 2, 2, M, prec, ctx)
    L = mp.tile_chol(t, overwrite_input=False).to_numpy()
    printed = np.array([[1, 0, 0, 0], [0.3678794, 0.9298735, 0, 0],
                        [0.3678795, 0.1159098, 0.9226211, 0],
                        [0.2431167, 0.2994405, 0.2641753, 0.8839915]])
    np.testing.assert_allclose(L, printed, atol=6e-8)
    Lref = ref.tile_chol(4, 2, np.array([[2, 1], [1, 2]]), M)
    np.testing.assert_allclose(L, Lref, rtol=1e-6, atol=1e-7)
    # the FP32-tile signature of the printout (0.3678795 vs dense 0.3678794)
    assert abs(L[2, 0] - 0.3678795) < 5e-8
    # the input is untouched when overwrite_input = FALSE
    np.testing.assert_array_equal(t.to_numpy(), ref_round_grid(M, np.array([[2, 1], [1, 2]]), 2))


def test_paper_trsm_4x4(ctx, ref):
    """L X = I with B in single tiles."""
    import paper_2406_02701_b200 as mp

    M = paper_M()
    t = mp.MPCRTile(4, 4, 2, 2, M, [["double", "single"], ["single", "double"]], ctx)
    Lt = mp.tile_chol(t, overwrite_input=False)
    b = mp.MPCRTile(4, 4, 2, 2, np.eye(4), [["single", "single"], ["single", "single"]], ctx)
    mp.tile_trsm(Lt, b, "L", False, False, 1.0)
    X = b.to_numpy()
    printed = np.array([[1, 0, 0, 0], [-0.3956231, 1.075415, 0, 0],
                        [-0.3490305, -0.1351055, 1.083869, 0],
                        [-0.03670389, -0.3239073, -0.3239073, 1.131233]])
    np.testing.assert_allclose(X, printed, atol=1e-6)  # printed to 7 digits
    L = Lt.to_numpy()
    Xref = ref.tile_trsm(L, np.array([[2, 1], [1, 2]]), 2, np.eye(4), np.ones((2, 2), int),
                         (2, 2), False, False, False, 1.0)
    np.testing.assert_allclose(X, Xref, rtol=1e-6, atol=1e-7)


def test_paper_gemm_half(ctx):
    """PAPER.md:585-588 example: C = A*0 + 0.5*1 -> 0.5."""
    import paper_2406_02701_b200 as mp

    A = np.arange(1, 25, dtype=float).reshape((4, 6), order="F")
    a = mp.MPCRTile(4, 6, 2, 6, A, [["single"], ["single"]], ctx)
    b = mp.MPCRTile(6, 1, 6, 1, np.zeros((6, 1)), [["single"]], ctx)
    c = mp.MPCRTile(4, 1, 2, 1, np.ones((4, 1)), [["single"], ["single"]], ctx)
    mp.tile_gemm(a, b, c, False, False, 1.0, 0.5, num_threads=4)
    np.testing.assert_array_equal(c.to_numpy(), np.full((4, 1), 0.5))


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_tile_gemm_mixed(ctx, ref, rng, ta, tb):
    import paper_2406_02701_b200 as mp

    nb = 32
    A = rng.random((96, 64)) if not ta else rng.random((64, 96))
    B = rng.random((64, 128)) if not tb else rng.random((128, 64))
    Cm = rng.random((96, 128))
    gA = rng.integers(0, 3, (A.shape[0] // nb, A.shape[1] // nb))
    gB = rng.integers(0, 3, (B.shape[0] // nb, B.shape[1] // nb))
    gC = rng.integers(0, 3, (3, 4))
    a = mp.MPCRTile(*A.shape, nb, nb, A, gA, ctx)
    b = mp.MPCRTile(*B.shape, nb, nb, B, gB, ctx)
    c = mp.MPCRTile(96, 128, nb, nb, Cm, gC, ctx)
    mp.tile_gemm(a, b, c, ta, tb, 0.75, 0.25)
    want = ref.tile_gemm(a.to_numpy(), gA, (nb, nb), b.to_numpy(), gB, (nb, nb),
                         ref_round_grid(Cm, gC, nb), gC, (nb, nb), ta, tb, 0.75, 0.25)
    got = c.to_numpy()
    # tile-wise tolerance by destination precision
    for i in range(3):
        for j in range(4):
            g = got[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]
            w = want[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]
            tol = {0: 2e-3, 1: 1e-5, 2: 1e-13}[gC[i, j]]
            assert np.linalg.norm(g - w) <= tol * np.linalg.norm(w)


def ref_round_grid(M, grid, nb):
    from oracle.oracle import round_to

    out = M.copy()
    for i in range(grid.shape[0]):
        for j in range(grid.shape[1]):
            sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
            out[sl] = round_to(M[sl], int(grid[i, j]))
    return out


@pytest.mark.parametrize("side", ["L", "R"])
@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("trans", [False, True])
def test_tile_trsm_general(ctx, ref, rng, side, upper, trans):
    import paper_2406_02701_b200 as mp

    n, nb = 96, 32
    B0 = rng.random((n, n))
    L0 = np.linalg.cholesky(B0.T @ B0 + n * np.eye(n))
    T0 = L0.T if upper else L0
    gA = np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]])
    a = mp.MPCRTile(n, n, nb, nb, T0, gA, ctx)
    Bm = rng.random((n, 64)) if side == "L" else rng.random((64, n))
    gB = np.ones((3, 2), int) * 2 if side == "L" else np.ones((2, 3), int) * 2
    gB[0, 0] = 1
    b = mp.MPCRTile(*Bm.shape, nb, nb, Bm, gB, ctx)
    mp.tile_trsm(a, b, side, upper, trans, 2.0)
    want = ref.tile_trsm(a.to_numpy(), gA, nb, ref_round_grid(Bm, gB, nb), gB, (nb, nb),
                         side == "R", upper, trans, 2.0)
    got = b.to_numpy()
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)


def band_map(nt, b64=1, b32=2):
    g = np.zeros((nt, nt), int)
    for i in range(nt):
        for j in range(nt):
            d = abs(i - j)
            g[i, j] = 2 if d < b64 else (1 if d < b32 else 0)
    return g


@pytest.mark.parametrize("n,nb,b64,b32", [(512, 128, 1, 2), (1024, 128, 1, 3),
                                         (1024, 256, 1, 2), (768, 64, 2, 4),
                                         (1024, 128, 0, 0), (1024, 128, 9, 9)])
def test_tile_chol_matern_vs_oracle(ctx, ref, n, nb, b64, b32):
    """Mixed-precision tiled Cholesky vs the composed reference oracle on an
    exponential (Matern 0.5, range 0.1) covariance; relFrob(L) and logdet."""
    import paper_2406_02701_b200 as mp

    side = int(np.ceil(np.sqrt(n)))
    cov = ref.grid_matern(side, n, 0.5, 0.1, 1.0, 2)
    nt = n // nb
    g = band_map(nt, b64, b32)
    if b64 == 0:  # all-half except an FP32 diagonal: harsher
        g = np.where(np.eye(nt) > 0, 1, 0)
    t = mp.MPCRTile(n, n, nb, nb, cov, g, ctx)
    mp.tile_chol(t)
    L = t.to_numpy()
    Lref = ref.tile_chol(n, nb, g, cov)
    err = np.linalg.norm(L - Lref) / np.linalg.norm(Lref)
    dense = np.linalg.cholesky(cov)
    err_dense = np.linalg.norm(Lref - dense) / np.linalg.norm(dense)
    # the GPU factor is as close to the oracle as the oracle is to exact FP64
    # (same mixed-precision rounding budget), with a floor at FP64 level
    assert err <= max(4 * err_dense, 1e-12), (err, err_dense)
    ld = t.logdet()
    ld_ref = 2 * np.log(np.diag(Lref)).sum()
    assert abs(ld - ld_ref) <= max(4 * abs(2 * np.log(np.diag(dense)).sum() - ld_ref), 1e-10 * abs(ld_ref))
    assert np.all(np.triu(L, 1) == 0)


def test_tile_chol_not_pd(ctx):
    import paper_2406_02701_b200 as mp

    n, nb = 256, 64
    M = np.eye(n)
    M[150, 150] = -2.0
    t = mp.MPCRTile(n, n, nb, nb, M, np.full((4, 4), 2), ctx)
    with pytest.raises(mp.MPError) as e:
        mp.tile_chol(t)
    assert e.value.kind == "NotPositiveDefinite" and e.value.info == 150


def test_tile_fill_matern_matches_reference(ctx, ref):
    import paper_2406_02701_b200 as mp

    n, nb, side = 300, 60, 18
    g = band_map(5, 1, 2)
    t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    t.fill_matern(side, 0.5, 0.1, 1.0)
    got = t.to_numpy()
    want = ref_round_grid(ref.grid_matern(side, n, 0.5, 0.1, 1.0, 2), g, nb)
    np.testing.assert_allclose(got, want, rtol=2e-15, atol=0)
    for nu in (1.5, 2.5):
        t.fill_matern(side, nu, 0.2, 2.0)
        want = ref_round_grid(ref.grid_matern(side, n, nu, 0.2, 2.0, 2), g, nb)
        # half tiles may straddle a rounding boundary by 1 ulp of half
        np.testing.assert_allclose(t.to_numpy(), want, rtol=2.0 ** -10, atol=0)


def test_get_tile_view(ctx):
    import paper_2406_02701_b200 as mp

    M = np.arange(64, dtype=float).reshape((8, 8), order="F")
    t = mp.MPCRTile(8, 8, 4, 4, M, [["double", "single"], ["half", "double"]], ctx)
    v = t.GetTile(2, 1)
    assert v.precision() == mp.Precision.Half
    np.testing.assert_array_equal(v.to_numpy(), M[4:8, 0:4])
    with pytest.raises(mp.MPError):
        t.GetTile(3, 1)


def test_dist_world1_matches_single(ctx, ref):
    """The distributed executor on a 1 x 1 process grid runs the same plan as
    the single-GPU path: identical factor, logdet and nll; NCCL resolves."""
    import paper_2406_02701_b200 as mp

    assert len(mp.nccl_unique_id()) == 128
    n, nb = 1024, 128
    side = 32
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    grid = mp.ProcessGrid(0, 1, 1, 1, ctx=ctx)
    a = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    b = mp.MPCRTile(n, n, nb, nb, None, g, grid=grid)
    assert b.owns(3, 1) and b.owns(2, 2) and not b.owns(1, 3)
    for t in (a, b):
        t.fill_matern(side, 0.5, 0.03, 1.0)
    mp.tile_chol(a)
    mp.tile_chol(b)
    La, Lb = a.to_numpy(), b.to_numpy()
    assert np.array_equal(La, Lb)
    assert a.logdet() == b.logdet()
    cov = ref.grid_matern(side, n, 0.5, 0.03, 1.0, 2)
    want = ref.tile_chol(n, nb, g, cov)
    dense = np.linalg.cholesky(ref_round_grid(cov, g, nb))
    err = np.linalg.norm(Lb - want) / np.linalg.norm(want)
    err_dense = np.linalg.norm(want - dense) / np.linalg.norm(dense)
    assert err <= max(4 * err_dense, 1e-12), (err, err_dense)



def test_tile_chol_graph_replay_bitwise(ctx):
    """First chol runs eagerly, the second is captured as a CUDA graph, later
    ones replay it: all factors identical bit for bit, launches counted."""
    import paper_2406_02701_b200 as mp

    n, nb = 2048, 256
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    A0 = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    A0.fill_matern(64, 0.5, 0.03, 1.0)
    A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    outs, counts = [], []
    for _ in range(4):
        A.copy_from(A0)
        l0 = ctx.launch_count()
        mp.tile_chol(A)
        counts.append(ctx.launch_count() - l0)
        outs.append(A.to_numpy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert counts[2] == counts[3] > 0


def test_tile_fill_matern_points_half_bit_exact(ctx, ref):
    """fill_matern_points on FP16 tiles: the FP32 fast exponential must give
    exactly the reference's double value rounded by encode_f16 (covariance.cpp
    + precision.cpp:49-93), nugget on the diagonal included."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    rng = np.random.default_rng(11)
    n, nb = 2048, 256  # 12.6 M half values over the three parameter sets
    x = rng.random(n)
    y = rng.random(n)
    d = np.hypot(x[:, None] - x[None], y[:, None] - y[None])
    for rng_a, var, nug in ((0.03, 1.0, 0.0), (0.1, 2.0, 0.25), (0.5, 0.75, 0.0)):
        g = np.zeros((n // nb, n // nb), int)  # all FP16
        t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
        t.fill_matern_points(x, y, 0.5, rng_a, var, nug)
        want = var * np.exp(-d / rng_a) + nug * np.eye(n)
        np.testing.assert_array_equal(t.to_numpy(), round_to(want, 0))


def test_tile_fill_matern_points_half_narrow_strips(ctx, ref):
    """The same bit-exactness for a tile size that is a multiple of 32 but not
    of 128 (the generator's one-block strips) and for 128-multiples
    (four-block strips), upper tiles included."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    rng = np.random.default_rng(5)
    for n, nb in ((960, 96), (1024, 128)):
        x = rng.random(n)
        y = rng.random(n)
        d = np.hypot(x[:, None] - x[None], y[:, None] - y[None])
        g = np.zeros((n // nb, n // nb), int)
        t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
        t.fill_matern_points(x, y, 0.5, 0.05, 1.5, 0.1)
        want = 1.5 * np.exp(-d / 0.05) + 0.1 * np.eye(n)
        np.testing.assert_array_equal(t.to_numpy(), round_to(want, 0))


_ENV_PROBE = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
n, nb = 4096, 256
nt = n // nb
i, j = np.indices((nt, nt))
g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A.fill_matern(64, 0.5, 0.03, 1.0)
mp.tile_chol(A)
print(hashlib.sha256(np.ascontiguousarray(A.to_numpy()).tobytes()).hexdigest())
"""


@pytest.mark.parametrize("env", [{"MPCR_UPDATE_GROUP": "1"}, {"MPCR_UPDATE_GROUP": "3"},
                                 {"MPCR_TC2_STAGES": "5"}, {"MPCR_LOOKAHEAD": "0"},
                                 {"MPCR_WB_ASYNC": "1"}])
def test_tile_chol_schedule_knobs_bitwise(env):
    """Update-tile order (MPCR_UPDATE_GROUP), the pair kernel's stage count and
    the lookahead and the write-back stream (MPCR_WB_ASYNC) change only the schedule, never the arithmetic: the factor
    is bit-identical to the default run (16 x 16 tiles, 2 update groups)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(extra):
        e = dict(os.environ)
        for k in ("MPCR_UPDATE_GROUP", "MPCR_TC2_STAGES", "MPCR_LOOKAHEAD", "MPCR_WB_ASYNC"):
            e.pop(k, None)
        e.update(extra)
        out = subprocess.run([sys.executable, "-c", _ENV_PROBE, root], env=e, capture_output=True,
                             text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        return out.stdout.strip().splitlines()[-1]

    assert run(env) == run({})


def test_tile_chol_graph_survives_scratch_growth(ctx):
    """The captured factorization graph bakes in context scratch pointers
    (POTRF barriers / leaf inverses in slot 1, 3xTF32 splits in slot 2).
    Growing those slots between chols (array uploads, an FP32 GEMM, a large
    row gather) must invalidate and re-capture the graph: the factors stay
    bit-identical and nothing writes freed memory."""
    import paper_2406_02701_b200 as mp

    n, nb = 2048, 256
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) < 3, 1, 0))  # FP32 head + tail tiles
    A0 = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    A0.fill_matern(64, 0.5, 0.03, 1.0)
    A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    outs = []
    for it in range(5):
        A.copy_from(A0)
        mp.tile_chol(A)
        outs.append(A.to_numpy())
        if it >= 1:  # grow scratch slots 1 and 2 after the graph exists
            m = 1024 * (it + 2)
            big = mp.MPArray.from_numpy(np.ones((m, m)), mp.Precision.Single, ctx)
            c = mp.MPArray.zeros_matrix(m, m, mp.Precision.Single, ctx)
            mp.linalg.gemm(big, big, c)
            A0.get_rows(np.arange(0, n, 3))
            ctx.synchronize()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_tile_chol_linv_generations_bitwise():
    """Wide FP64/FP32 bands put FP64 and FP32 tiles in the tail TRSM of every
    panel, which reads Linv_k on the lookahead stream while the next step's
    POTRF/TRTRI writes Linv_{k+1}: with two Linv generations the factor equals
    the serial (MPCR_LOOKAHEAD=0) one bit for bit."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    probe = r'''
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
n, nb = 8192, 512
nt = n // nb
i, j = np.indices((nt, nt))
g = np.where(abs(i - j) < 3, 2, np.where(abs(i - j) < 5, 1, 0))
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A.fill_matern(91, 0.5, 0.03, 1.0)
for _ in range(3):  # eager, captured, replayed
    B = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    B.copy_from(A)
    mp.tile_chol(B)
print(hashlib.sha256(np.ascontiguousarray(B.to_numpy()).tobytes()).hexdigest())
'''

    def run(extra):
        e = dict(os.environ)
        e.pop("MPCR_LOOKAHEAD", None)
        e.update(extra)
        out = subprocess.run([sys.executable, "-c", probe, root], env=e, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return out.stdout.strip().splitlines()[-1]

    assert run({}) == run({"MPCR_LOOKAHEAD": "0"})


_PAIR_PROBE = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
n, nb = 4096, 512
nt = n // nb
i, j = np.indices((nt, nt))
g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A.fill_matern(64, 0.5, 0.03, 1.0)
mp.tile_chol(A)
np.save(sys.argv[2], A.to_numpy())
"""


def test_paired_steps_match_unpaired_within_rounding(ctx, ref, tmp_path):
    """Paired steps (default) apply two panels to a tile in one pass and round
    once; MPCR_PAIR_STEPS=0 rounds after every step.  Both are checked against
    the composed reference oracle with the 4x rule."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for v in ("1", "0"):
        f = tmp_path / f"L{v}.npy"
        e = dict(os.environ, MPCR_PAIR_STEPS=v)
        r = subprocess.run([sys.executable, "-c", _PAIR_PROBE, root, str(f)], env=e, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[v] = np.load(f)
    n, nb = 4096, 512
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    cov = ref.grid_matern(64, n, 0.5, 0.03, 1.0, 2)
    Lref = ref.tile_chol(n, nb, g, cov)
    dense = np.linalg.cholesky(ref_round_grid(cov, g, nb))
    err_dense = np.linalg.norm(Lref - dense) / np.linalg.norm(dense)
    for v, L in outs.items():
        err = np.linalg.norm(L - Lref) / np.linalg.norm(Lref)
        assert err <= 4 * err_dense, (v, err, err_dense)
    assert not np.array_equal(outs["1"], outs["0"])  # the pairing is really on by default


_OZ32_PROBE = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
n, nb = 4096, 512
nt = n // nb
i, j = np.indices((nt, nt))
g = np.where(i == j, 2, np.where(abs(i - j) < 4, 1, 0))
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A.fill_matern(64, 0.5, 0.03, 1.0)
ctx.prof_enable(True)
mp.tile_chol(A)
ctx.synchronize()
print("int8_launches", ctx.prof_query(7)[1])
np.save(sys.argv[2], A.to_numpy())
"""


def test_fp32_band_on_int8_digits_matches_oracle(ctx, ref, tmp_path):
    """FP32 tiles fed by FP32 panel tiles (an FP32 band of width 4, SURVEY
    §8d's example) run on INT8 digits by default (digits exact to 2^-41 of
    each row's maximum, FP64 combination, one rounding to FP32) and on DMMA
    with MPCR_OZAKI32=0.  Both factors satisfy the 4x oracle rule and differ
    from each other by less than the oracle differs from FP64."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs, i8 = {}, {}
    for v in ("1", "0"):
        f = tmp_path / f"L{v}.npy"
        e = dict(os.environ, MPCR_OZAKI32=v)
        r = subprocess.run([sys.executable, "-c", _OZ32_PROBE, root, str(f)], env=e, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[v] = np.load(f)
        i8[v] = int(r.stdout.split("int8_launches")[1].split()[0])
    assert i8["1"] > i8["0"], i8  # the FP32 band really runs on the INT8 kernel by default
    n, nb = 4096, 512
    nt = n // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) < 4, 1, 0))
    cov = ref.grid_matern(64, n, 0.5, 0.03, 1.0, 2)
    Lref = ref.tile_chol(n, nb, g, cov)
    dense = np.linalg.cholesky(ref_round_grid(cov, g, nb))
    err_dense = np.linalg.norm(Lref - dense) / np.linalg.norm(dense)
    for v, L in outs.items():
        err = np.linalg.norm(L - Lref) / np.linalg.norm(Lref)
        assert err <= 4 * err_dense, (v, err, err_dense)
    d = np.linalg.norm(outs["1"] - outs["0"]) / np.linalg.norm(outs["0"])
    assert d <= err_dense, d
