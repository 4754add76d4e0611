"""GPU parity: dense kernels (linalg.hpp:23-54) vs the reference oracle.

Tolerances (north star: normwise relative error <= c * n * u_p):
GEMM family rel. Frobenius error <= 4 * k * u(compute precision); Cholesky
factors <= 100 * n * u; exact cases (A*I, symmetry, beta-only,
error codes) are exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, S, D = 0, 1, 2
U = {H: 2.0 ** -24, S: 2.0 ** -24, D: 2.0 ** -53}  # compute precision roundoff
UST = {H: 2.0 ** -11, S: 2.0 ** -24, D: 2.0 ** -53}  # storage roundoff


def rel(a, b):
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


def gemm_tol(k, pc):
    return 4 * max(k, 1) * U[pc] + 2 * UST[pc]


def mk(rng, shape, p):
    from oracle.oracle import round_to

    return round_to(rng.random(shape), p)


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("pc", [H, S, D])
def test_gemm_trans_precisions(ctx, ref, rng, ta, tb, pc):
    import paper_2406_02701_b200 as mp

    m, n, k = 67, 45, 33
    for pa in range(pc + 1):
        for pb in range(pc + 1):
            A = mk(rng, (k, m) if ta else (m, k), pa)
            B = mk(rng, (n, k) if tb else (k, n), pb)
            Cm = mk(rng, (m, n), pc)
            for alpha, beta in ((1.0, 0.0), (0.7, 0.3), (-1.0, 1.0)):
                da = mp.MPArray.from_numpy(A, mp.Precision(pa), ctx)
                db = mp.MPArray.from_numpy(B, mp.Precision(pb), ctx)
                dc = mp.MPArray.from_numpy(Cm, mp.Precision(pc), ctx)
                mp.linalg.gemm(da, db, dc, ta, tb, alpha, beta)
                want = ref.gemm(pa, pb, pc, A, B, Cm, ta, tb, alpha, beta)
                assert rel(dc.to_numpy(), want) <= gemm_tol(k, pc)


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("pc", [H, S])
def test_gemm_fp16_tensor_core(ctx, ref, rng, ta, tb, pc):
    """Half x half -> half/single runs on tcgen05 (shapes with ragged edges)."""
    import paper_2406_02701_b200 as mp

    for (m, n, k) in ((256, 256, 64), (384, 512, 320), (200, 300, 136), (128, 1000, 1000)):
        A = mk(rng, (k, m) if ta else (m, k), H) - 0.5
        B = mk(rng, (n, k) if tb else (k, n), H) - 0.5
        Cm = mk(rng, (m, n), pc)
        da = mp.MPArray.from_numpy(A, mp.Precision.Half, ctx)
        db = mp.MPArray.from_numpy(B, mp.Precision.Half, ctx)
        dc = mp.MPArray.from_numpy(Cm, mp.Precision(pc), ctx)
        mp.linalg.gemm(da, db, dc, ta, tb, -1.0, 1.0)
        want = ref.gemm(H, H, pc, A, B, Cm, ta, tb, -1.0, 1.0)
        err = rel(dc.to_numpy(), want)
        assert err <= gemm_tol(k, pc), (m, n, k, err)


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_single_3xtf32(ctx, ref, rng, ta, tb):
    """Single C with half/single operands runs 3xTF32 on tcgen05; it must stay
    within the FP32 tolerance of the reference's float GEMM."""
    import paper_2406_02701_b200 as mp

    for (m, n, k) in ((256, 256, 64), (384, 512, 320), (200, 300, 136), (1024, 512, 1000)):
        for pa, pb in ((S, S), (H, S), (S, H)):
            A = mk(rng, (k, m) if ta else (m, k), pa) - 0.5
            B = mk(rng, (n, k) if tb else (k, n), pb) - 0.5
            Cm = mk(rng, (m, n), S)
            da = mp.MPArray.from_numpy(A, mp.Precision(pa), ctx)
            db = mp.MPArray.from_numpy(B, mp.Precision(pb), ctx)
            dc = mp.MPArray.from_numpy(Cm, mp.Precision.Single, ctx)
            mp.linalg.gemm(da, db, dc, ta, tb, 0.5, -1.0)
            want = ref.gemm(pa, pb, S, A, B, Cm, ta, tb, 0.5, -1.0)
            err = rel(dc.to_numpy(), want)
            assert err <= gemm_tol(k, S), (m, n, k, pa, pb, err)


def test_gemm_fp16_large_vs_fp64(ctx, rng):
    """n=2048 half GEMM against an exact FP64 product of the same halves."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    n = 2048
    A = round_to(rng.random((n, n)), H)
    B = round_to(rng.random((n, n)), H)
    da = mp.MPArray.from_numpy(A, mp.Precision.Half, ctx)
    db = mp.MPArray.from_numpy(B, mp.Precision.Half, ctx)
    dc = mp.MPArray.zeros_matrix(n, n, mp.Precision.Single, ctx)
    mp.linalg.gemm(da, db, dc)
    exact = A @ B
    # the tensor core's FP32 accumulator truncates (measured bias ~1e-5 at
    # k=2048); still inside the reference's k*u_single bound (1.2e-4)
    assert rel(dc.to_numpy(), exact) < 2048 * 2.0 ** -24
    dh = mp.MPArray.zeros_matrix(n, n, mp.Precision.Half, ctx)
    mp.linalg.gemm(da, db, dh)
    assert rel(dh.to_numpy(), exact) < 2 * 2.0 ** -11


def test_gemm_exact_cases(ctx, rng):
    """test_linalg.cpp:152-183: A*I = A exactly (double; half on the FP16
    tensor cores is exact too; single runs 3xTF32 and is exact to ~2^-22),
    beta-only, PrecisionMismatch."""
    import paper_2406_02701_b200 as mp

    for p in (H, S, D):
        A = mk(rng, (256, 256), p)
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        eye = mp.MPArray.from_numpy(np.eye(256), mp.Precision(p), ctx)
        dc = mp.MPArray.zeros_matrix(256, 256, mp.Precision(p), ctx)
        mp.linalg.gemm(da, eye, dc)
        if p == S:
            np.testing.assert_allclose(dc.to_numpy(), A, rtol=2.0 ** -21, atol=0)
        else:
            np.testing.assert_array_equal(dc.to_numpy(), A)
    a = mp.MPArray.from_numpy(mk(rng, (3, 3), D), mp.Precision.Double, ctx)
    zero = mp.MPArray.zeros_matrix(3, 3, mp.Precision.Double, ctx)
    ones = mp.MPArray.from_numpy(np.ones((3, 3)), mp.Precision.Double, ctx)
    mp.linalg.gemm(a, zero, ones, False, False, 1.0, 0.5)
    np.testing.assert_array_equal(ones.to_numpy(), np.full((3, 3), 0.5))
    low = mp.MPArray.zeros_matrix(3, 3, mp.Precision.Single, ctx)
    with pytest.raises(mp.MPError) as e:
        mp.linalg.gemm(a, a, low)
    assert e.value.kind == "PrecisionMismatch"
    with pytest.raises(mp.MPError) as e:
        mp.linalg.gemm(a, mp.MPArray.zeros_matrix(4, 4, mp.Precision.Double, ctx), zero)
    assert e.value.kind == "ShapeMismatch"


def test_matmul_crossprod(ctx, ref, rng):
    import paper_2406_02701_b200 as mp

    for pa in (H, S, D):
        for pb in (H, S, D):
            A = mk(rng, (40, 30), pa)
            B = mk(rng, (30, 20), pb)
            da = mp.MPArray.from_numpy(A, mp.Precision(pa), ctx)
            db = mp.MPArray.from_numpy(B, mp.Precision(pb), ctx)
            out = mp.linalg.matmul(da, db)
            assert out.precision() == max(pa, pb)
            pc = max(pa, pb)
            assert rel(out.to_numpy(), ref.matmul(pa, pb, A, B)) <= gemm_tol(30, pc)
    for p in (H, S, D):
        for n in (5, 300):
            A = mk(rng, (n + 7, n), p)
            da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
            c = mp.linalg.crossprod(da).to_numpy()
            np.testing.assert_array_equal(c, c.T)  # exactly symmetric (test_linalg.cpp:132-135)
            assert rel(c, ref.crossprod(p, A)) <= gemm_tol(n + 7, p)


def test_crossprod_error_bands_1024(ctx, ref):
    """acceptance.cpp:153-177 criterion 4 at n=1024 on the reference's inputs."""
    import paper_2406_02701_b200 as mp

    n = 1024
    A = ref.rng_uniform(1000 + n, n * n).reshape((n, n), order="F")
    oracle = ref.crossprod(D, A)
    errs = {}
    for p in (H, S, D):
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        errs[p] = rel(mp.linalg.crossprod(da).to_numpy(), oracle)
    assert 1e-4 <= errs[H] <= 2e-2
    assert 1e-8 <= errs[S] <= 1e-5
    assert errs[D] <= 1e-13
    assert errs[H] > errs[S] > errs[D]


def spd(rng, n):
    B = rng.random((n, n))
    return B.T @ B + n * np.eye(n)


@pytest.mark.parametrize("n", [1, 2, 8, 63, 64, 65, 200, 1024])
def test_chol(ctx, ref, rng, n):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    A0 = spd(rng, n)
    for p in (H, S, D):
        A = round_to(A0, p)
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        U = mp.linalg.chol(da).to_numpy()
        Uref = ref.chol(p, A)
        assert np.all(np.tril(U, -1) == 0)
        tol = 100 * n * (2.0 ** -24 if p != D else 2.0 ** -53) + 2 * UST[p]
        assert rel(U, Uref) <= tol, (p, rel(U, Uref))


def test_chol_known_and_failures(ctx):
    """test_linalg.cpp:185-221."""
    import paper_2406_02701_b200 as mp

    a = mp.MPArray.from_doubles([4, 2, 2, 3], 2, 2, mp.Precision.Double, ctx)
    u = mp.linalg.chol(a).to_numpy()
    assert u[0, 0] == 2.0 and u[0, 1] == 1.0 and u[1, 0] == 0.0
    assert abs(u[1, 1] - np.sqrt(2.0)) < 1e-15
    eye = mp.MPArray.from_numpy(np.eye(4), mp.Precision.Double, ctx)
    np.testing.assert_array_equal(mp.linalg.chol(eye).to_numpy(), np.eye(4))
    bad = mp.MPArray.from_doubles([1, 2, 2, 1], 2, 2, mp.Precision.Double, ctx)
    with pytest.raises(mp.MPError) as e:
        mp.linalg.chol(bad)
    assert e.value.kind == "NotPositiveDefinite" and e.value.info == 1
    neg = mp.MPArray.from_doubles([-1.0], 1, 1, mp.Precision.Double, ctx)
    with pytest.raises(mp.MPError) as e:
        mp.linalg.chol(neg)
    assert e.value.info == 0
    # a failing pivot deep inside a blocked factorization
    n = 300
    M = np.eye(n)
    M[200, 200] = -1.0
    with pytest.raises(mp.MPError) as e:
        mp.linalg.chol(mp.MPArray.from_numpy(M, mp.Precision.Double, ctx))
    assert e.value.info == 200
    with pytest.raises(mp.MPError) as e:
        mp.linalg.chol(mp.MPArray.zeros_matrix(2, 3, mp.Precision.Double, ctx))
    assert e.value.kind == "ShapeMismatch"


def test_chol_reads_upper_triangle(ctx, ref, rng):
    """chol_kernel reads the upper triangle only (linalg.cpp:110-127)."""
    import paper_2406_02701_b200 as mp

    A = spd(rng, 50)
    A[np.tril_indices(50, -1)] = 7.0  # garbage below the diagonal
    da = mp.MPArray.from_numpy(A, mp.Precision.Double, ctx)
    assert rel(mp.linalg.chol(da).to_numpy(), ref.chol(D, A)) < 1e-13


@pytest.mark.parametrize("side_right", [False, True])
@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("trans", [False, True])
def test_trsm(ctx, ref, rng, side_right, upper, trans):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    n = 48
    U0 = np.linalg.cholesky(spd(rng, n)).T
    T0 = U0 if upper else U0.T
    for pa in (H, S, D):
        for pb in (H, S, D):
            T = round_to(T0, pa)
            B = round_to(rng.random((7, n) if side_right else (n, 7)), pb)
            da = mp.MPArray.from_numpy(T, mp.Precision(pa), ctx)
            db = mp.MPArray.from_numpy(B, mp.Precision(pb), ctx)
            mp.linalg.trsm(da, db, mp.Side(int(side_right)), upper, trans, 1.5)
            want = ref.trsm(pa, pb, T, B, side_right, upper, trans, 1.5)
            tol = 100 * n * U[pb] + 2 * UST[pb]
            assert rel(db.to_numpy(), want) <= tol


def test_trsm_singular_and_solves(ctx, ref, rng):
    import paper_2406_02701_b200 as mp

    z = np.eye(3)
    z[2, 2] = 0.0
    dz = mp.MPArray.from_numpy(z, mp.Precision.Double, ctx)
    b = mp.MPArray.from_numpy(rng.random((3, 1)), mp.Precision.Double, ctx)
    with pytest.raises(mp.MPError) as e:
        mp.linalg.backsolve(dz, b)
    assert e.value.kind == "SingularMatrix"
    L = np.linalg.cholesky(spd(rng, 20))
    B = rng.random((20, 3))
    for pt in (S, D):
        for pb in (S, D):
            from oracle.oracle import round_to

            Lr, Br = round_to(L, pt), round_to(B, pb)
            dl = mp.MPArray.from_numpy(Lr, mp.Precision(pt), ctx)
            db = mp.MPArray.from_numpy(Br, mp.Precision(pb), ctx)
            f = mp.linalg.forwardsolve(dl, db)
            assert rel(f.to_numpy(), ref.trisolve(False, pt, pb, Lr, Br)) < 1e-5
            du = mp.MPArray.from_numpy(Lr.T.copy(), mp.Precision(pt), ctx)
            g = mp.linalg.backsolve(du, db)
            assert rel(g.to_numpy(), ref.trisolve(True, pt, pb, Lr.T, Br)) < 1e-5


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_half_to_double_int8_digits(ctx, rng, ta, tb):
    """FP16 x FP16 -> FP64 runs on the INT8 tensor cores with exact 7-bit
    digit slicing (ozaki.cu): every digit product is exact, so against an
    extended-precision sum of the exact FP16 products the error is a few FP64
    roundings of the result, over a 2^-24 .. 2^14 dynamic range."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    for (m, n, k) in ((256, 256, 1024), (300, 200, 700), (67, 45, 33)):
        def wide(shape):
            v = rng.standard_normal(shape) * np.exp2(rng.integers(-20, 12, size=shape))
            return round_to(v, H)
        A = wide((k, m) if ta else (m, k))
        B = wide((n, k) if tb else (k, n))
        Cm = rng.standard_normal((m, n))
        opA = A.T if ta else A
        opB = B.T if tb else B
        exact = opA.astype(np.longdouble) @ opB.astype(np.longdouble)
        want = (-1.0 * exact + Cm.astype(np.longdouble))
        da = mp.MPArray.from_numpy(A, mp.Precision.Half, ctx)
        db = mp.MPArray.from_numpy(B, mp.Precision.Half, ctx)
        dc = mp.MPArray.from_numpy(Cm, mp.Precision.Double, ctx)
        mp.linalg.gemm(da, db, dc, ta, tb, -1.0, 1.0)
        got = dc.to_numpy()
        scale = np.abs(opA) @ np.abs(opB) + np.abs(Cm)
        err = np.abs(got.astype(np.longdouble) - want) / scale
        assert err.max() <= 16 * 2.0 ** -53, (m, n, k, float(err.max()))


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_gemm_half_to_double_large_k_chunks(ctx, ta, tb):
    """K beyond the int32-exact limit of one digit group (6 K 64^2 < 2^31):
    the INT8-digit path splits K into OZ_MAX_K = 65536 chunks summed in FP64.
    All-positive near-maximal digits make every group sum as large as it can
    get; an unchunked K = 2^19 + 96 would overflow the single-pair group."""
    import paper_2406_02701_b200 as mp

    m, n, k = 64, 32, (1 << 19) + 96
    r = np.random.default_rng(3)
    A = (1.0 + r.integers(0, 1024, (m, k)) / 1024.0).astype(np.float16).astype(np.float64)
    B = (1.0 + r.integers(0, 1024, (k, n)) / 1024.0).astype(np.float16).astype(np.float64)
    A[:, 0] = 1.9990234375  # row maxima just below 2: leading digits near 64
    A_st = np.asfortranarray(A.T) if ta else A
    B_st = np.asfortranarray(B.T) if tb else B
    da = mp.MPArray.from_numpy(A_st, mp.Precision.Half, ctx)
    db = mp.MPArray.from_numpy(B_st, mp.Precision.Half, ctx)
    dc = mp.MPArray.zeros_matrix(m, n, mp.Precision.Double, ctx)
    mp.linalg.gemm(da, db, dc, ta, tb, 1.0, 0.0)
    got = dc.to_numpy()
    exact = A.astype(np.longdouble) @ B.astype(np.longdouble)
    err = np.abs(got.astype(np.longdouble) - exact) / exact
    assert err.max() <= 16 * 2.0 ** -53, float(err.max())


def test_gemm_half_to_double_block_digit_counts(ctx):
    """Digit counts are kept per 128-row block and the slicer writes only the
    planes a block needs: blocks of one operand needing 1, 2, .. 6 digits (and
    an all-zero block), after a call that filled every plane of the same
    scratch with nonzero digits -- the stale planes must never be read."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    r = np.random.default_rng(11)
    m, n, k = 896, 256, 512
    # warm-up: every row spans 2^-24 .. 2^5 -> six digits in every block
    W = round_to(r.standard_normal((m, k)) * np.exp2(r.integers(-24, 5, size=(m, k))), H)
    dw = mp.MPArray.from_numpy(W, mp.Precision.Half, ctx)
    dwb = mp.MPArray.from_numpy(W[:n].T.copy(), mp.Precision.Half, ctx)
    dc0 = mp.MPArray.zeros_matrix(m, n, mp.Precision.Double, ctx)
    mp.linalg.gemm(dw, dwb, dc0)
    # block b of A: dynamic range growing with b (block 6 all zero)
    A = np.zeros((m, k))
    for b in range(7):
        rows = slice(b * 128, (b + 1) * 128)
        if b == 6:
            continue
        span = 1 + 7 * b  # binades
        A[rows] = r.standard_normal((128, k)) * np.exp2(-r.integers(0, span, size=(128, k)))
    A = round_to(A, H)
    B = round_to(r.standard_normal((k, n)), H)
    da = mp.MPArray.from_numpy(A, mp.Precision.Half, ctx)
    db = mp.MPArray.from_numpy(B, mp.Precision.Half, ctx)
    dc = mp.MPArray.zeros_matrix(m, n, mp.Precision.Double, ctx)
    mp.linalg.gemm(da, db, dc)
    got = dc.to_numpy()
    exact = A.astype(np.longdouble) @ B.astype(np.longdouble)
    scale = np.abs(A) @ np.abs(B)
    err = np.abs(got.astype(np.longdouble) - exact) / np.where(scale > 0, scale, 1.0)
    assert err.max() <= 16 * 2.0 ** -53, float(err.max())
    assert np.all(got[768:] == 0.0)


def test_gemm_half_to_double_nonfinite(ctx):
    """Inf/NaN in an FP16 operand row propagate as NaN to that output row."""
    import paper_2406_02701_b200 as mp

    A = np.ones((128, 64))
    A[5, 3] = np.inf
    B = np.ones((64, 128))
    da = mp.MPArray.from_numpy(A, mp.Precision.Half, ctx)
    db = mp.MPArray.from_numpy(B, mp.Precision.Half, ctx)
    dc = mp.MPArray.from_numpy(np.zeros((128, 128)), mp.Precision.Double, ctx)
    mp.linalg.gemm(da, db, dc)
    got = dc.to_numpy()
    assert np.isnan(got[5]).all() or np.isinf(got[5]).all()
    assert np.all(got[np.arange(128) != 5] == 64.0)


@pytest.mark.parametrize("p", [S, D])
def test_solve_spd_and_lu_paths(ctx, ref, rng, p):
    """solve(a, b) (linalg.cpp:551-575): exactly symmetric SPD a takes the
    Cholesky path, a general a the LU path (partial pivoting); both against
    the reference's solve in the same precisions."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    n, k = 200, 7
    X = rng.standard_normal((n, n))
    spd = round_to(X @ X.T / n + np.eye(n), p)
    gen = round_to(rng.standard_normal((n, n)) + 0.1 * np.eye(n), p)  # pivoting happens
    B = round_to(rng.standard_normal((n, k)), p)
    for A in (spd, gen):
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        db = mp.MPArray.from_numpy(B, mp.Precision(p), ctx)
        got = mp.linalg.solve(da, db).to_numpy()
        want = ref.solve(p, p, A, B)
        cond = np.linalg.cond(A)
        tol = 16 * n * U[p] * cond
        assert rel(got, want) <= tol, (p, rel(got, want), tol)
    # inverse (b omitted) of the general matrix
    inv = mp.linalg.solve(mp.MPArray.from_numpy(gen, mp.Precision(p), ctx)).to_numpy()
    assert rel(inv, ref.solve(p, p, gen, np.eye(n))) <= 16 * n * U[p] * np.linalg.cond(gen)


def test_solve_lu_bit_exact_factors(ctx, ref, rng):
    """The LU path follows lu_kernel's operation order (first maximal pivot,
    IEEE division, separate multiply and subtract): on a small matrix with
    many ties and a permutation-heavy pattern the FP64 solution equals the
    reference's to the last bit or within a few ulps (substitution order)."""
    import paper_2406_02701_b200 as mp

    n = 48
    A = np.round(rng.standard_normal((n, n)) * 4) / 4  # many equal magnitudes (ties)
    A += np.diag(np.where(np.arange(n) % 3 == 0, 0.0, 0.5))
    B = rng.standard_normal((n, 2))
    got = mp.linalg.solve(mp.MPArray.from_numpy(A, mp.Precision.Double, ctx),
                          mp.MPArray.from_numpy(B, mp.Precision.Double, ctx)).to_numpy()
    want = ref.solve(D, D, A, B)
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-12


def test_solve_errors(ctx):
    import paper_2406_02701_b200 as mp

    sing = np.ones((8, 8))
    with pytest.raises(mp.MPError) as e:
        mp.linalg.solve(mp.MPArray.from_numpy(sing, mp.Precision.Double, ctx),
                        mp.MPArray.from_numpy(np.ones((8, 1)), mp.Precision.Double, ctx))
    assert e.value.kind == "SingularMatrix"
    with pytest.raises(mp.MPError) as e:
        mp.linalg.solve(mp.MPArray.from_numpy(np.eye(8), mp.Precision.Double, ctx),
                        mp.MPArray.from_numpy(np.ones((7, 1)), mp.Precision.Double, ctx))
    assert e.value.kind == "ShapeMismatch"


@pytest.mark.parametrize("p", [S, D])
def test_chol2inv(ctx, ref, rng, p):
    """chol2inv (linalg.cpp:383-408): exactly symmetric (U^T U)^-1."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    n = 160
    X = rng.standard_normal((n, n))
    A = X @ X.T / n + np.eye(n)
    Uf = round_to(ref.chol(p, round_to(A, p)), p)
    got = mp.linalg.chol2inv(mp.MPArray.from_numpy(Uf, mp.Precision(p), ctx)).to_numpy()
    want = ref.chol2inv(p, Uf)
    assert np.array_equal(got, got.T)
    assert rel(got, want) <= 16 * n * U[p] * np.linalg.cond(A), rel(got, want)
    with pytest.raises(mp.MPError) as e:
        Z = Uf.copy()
        Z[5, 5] = 0.0
        mp.linalg.chol2inv(mp.MPArray.from_numpy(Z, mp.Precision(p), ctx))
    assert e.value.kind == "SingularMatrix"


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_double_small_split_k(ctx, rng, ta, tb):
    """FP64 DMMA launches that leave SMs idle split K over a cluster (2 or 4
    CTAs, DSMEM reduction in rank order): ragged shapes, both layouts,
    deterministic run to run."""
    import paper_2406_02701_b200 as mp

    for (m, n, k) in ((512, 512, 512), (130, 70, 1000), (64, 64, 4096), (200, 190, 130), (33, 17, 257)):
        A = rng.random((k, m) if ta else (m, k)) - 0.5
        B = rng.random((n, k) if tb else (k, n)) - 0.5
        C0 = rng.random((m, n))
        want = 0.5 * C0 - (A.T if ta else A) @ (B.T if tb else B)
        outs = []
        for _ in range(2):
            dc = mp.MPArray.from_numpy(C0, mp.Precision.Double, ctx)
            mp.linalg.gemm(mp.MPArray.from_numpy(A, mp.Precision.Double, ctx),
                           mp.MPArray.from_numpy(B, mp.Precision.Double, ctx), dc, ta, tb, -1.0, 0.5)
            outs.append(dc.to_numpy())
        assert rel(outs[0], want) <= gemm_tol(k, D), (m, n, k)
        np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n,bad", [(300, 64), (300, 127), (300, 128), (300, 130), (1000, 999), (1024, 16)])
def test_chol_failing_pivot_positions(ctx, n, bad):
    """NotPositiveDefinite reports the first failing column (errors.hpp:25-31)
    wherever it falls relative to the 64-blocks and 16-column panels."""
    import paper_2406_02701_b200 as mp

    M = np.eye(n) * 4.0
    M[bad, bad] = -1.0
    for p in (S, D):
        with pytest.raises(mp.MPError) as e:
            mp.linalg.chol(mp.MPArray.from_numpy(M, mp.Precision(p), ctx))
        assert e.value.kind == "NotPositiveDefinite" and e.value.info == bad, (p, e.value.info)


@pytest.mark.parametrize("prec", [H, S])
def test_gemm_grouped_rasterization_ragged(ctx, rng, prec):
    """Tile grids with more M-blocks than one rasterization group and a
    narrower last group (FP16 pair kernel: 8 pairs of 256 rows; 3xTF32
    single-CTA kernel: 16 blocks of 128 rows), ragged N and K."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    m, n, k = 4500, 700, 520
    A = round_to(rng.random((m, k)) - 0.5, prec)
    B = round_to(rng.random((n, k)) - 0.5, prec)
    da = mp.MPArray.from_numpy(A, mp.Precision(prec), ctx)
    db = mp.MPArray.from_numpy(B, mp.Precision(prec), ctx)
    dc = mp.MPArray.zeros_matrix(m, n, mp.Precision.Single, ctx)
    mp.linalg.gemm(da, db, dc, False, True, 1.0, 0.0)
    assert rel(dc.to_numpy(), A @ B.T) < 4 * k * 2.0 ** -24


@pytest.mark.parametrize("pa,pb", [(H, S), (S, D), (D, D), (H, H)])
def test_dispatch_registry_ops(ctx, ref, rng, pa, pb):
    """dispatch::resolve / execute (dispatch.cpp:46-137) by op name on device
    arrays: promoted keys, the same results as the reference's kernels
    (bit-exact for elementwise/concat/transpose, c*n*u for the rest)."""
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    m, n = 48, 48
    A = round_to(rng.random((m, n)) + 0.5, pa)
    B = round_to(rng.random((m, n)) + 0.5, pb)
    da, db = mp.MPArray.from_numpy(A, pa, ctx), mp.MPArray.from_numpy(B, pb, ctx)
    po = max(pa, pb)
    for i, op in enumerate(("add", "sub", "mul", "div")):
        key = mp.dispatch.resolve(op, pa, pb)
        assert (key.in_a, key.in_b, key.out) == (pa, pb, po) and not mp.dispatch.is_unary(op)
        got = mp.dispatch.execute(key, op, da, db)
        assert got.precision() == po
        np.testing.assert_array_equal(got.to_numpy(), ref.ew_binary(i, pa, pb, A, B))
    key = mp.dispatch.resolve("matmul", pa, pb)
    got = mp.dispatch.execute(key, "matmul", da, db).to_numpy()
    want = ref.matmul(pa, pb, A, B)
    assert np.linalg.norm(got - want) <= 4 * n * {0: 2.0 ** -11, 1: 2.0 ** -24, 2: 2.0 ** -53}[po] * np.linalg.norm(want) + 1e-300
    got = mp.dispatch.execute(mp.dispatch.resolve("crossprod", pa, pb), "crossprod", da, db).to_numpy()
    want = ref.crossprod(pa, A, pb, B)
    assert np.linalg.norm(got - want) <= 4 * m * {0: 2.0 ** -11, 1: 2.0 ** -24, 2: 2.0 ** -53}[po] * np.linalg.norm(want)
    for op, ax in (("rbind", 0), ("cbind", 1)):
        got = mp.dispatch.execute(mp.dispatch.resolve(op, pa, pb), op, da, db)
        np.testing.assert_array_equal(got.to_numpy(), np.concatenate([A, B], axis=ax))
    for i, op in enumerate(("log", "exp", "sqrt", "abs")):
        key = mp.dispatch.resolve(op, pa)
        assert key.in_b == -1 and key.out == pa and mp.dispatch.is_unary(op)
        got = mp.dispatch.execute(key, op, da).to_numpy()
        want = ref.ew_unary(i, pa, A)
        if op in ("sqrt", "abs"):
            np.testing.assert_array_equal(got, want)
        else:  # few-ulp
            np.testing.assert_allclose(got, want, rtol=4 * {0: 2.0 ** -11, 1: 2.0 ** -24, 2: 2.0 ** -52}[pa])
    np.testing.assert_array_equal(mp.dispatch.execute(mp.dispatch.resolve("transpose", pa), "transpose", da).to_numpy(),
                                  A.T)
    S_ = round_to(A.T @ A + m * np.eye(n), pa)
    dS = mp.MPArray.from_numpy(S_, pa, ctx)
    u = mp.dispatch.execute(mp.dispatch.resolve("chol", pa), "chol", dS).to_numpy()
    cp = max(pa, S)
    tol = 100 * n * {1: 2.0 ** -24, 2: 2.0 ** -53}[cp] + 2 * {0: 2.0 ** -11, 1: 2.0 ** -24, 2: 2.0 ** -53}[pa]
    uw = ref.chol(pa, S_)
    assert np.linalg.norm(u - uw) <= tol * np.linalg.norm(uw)
    inv = mp.dispatch.execute(mp.dispatch.resolve("solve", pa), "solve", dS).to_numpy()
    invw = ref.solve(pa, pa, S_, np.eye(n))
    assert np.linalg.norm(inv - invw) <= tol * np.linalg.norm(invw)
    # errors: unknown op, wrong precision for the key, arity
    with pytest.raises(mp.MPError) as e:
        mp.dispatch.resolve("qr", pa)
    assert e.value.kind == "UnknownOperation"
    with pytest.raises(mp.MPError) as e:
        mp.dispatch.execute(mp.dispatch.resolve("add", pb, pb), "add", da, db) if pa != pb else \
            mp.dispatch.execute(mp.dispatch.resolve("add", D if pa != D else H, pb), "add", da, db)
    assert e.value.kind == "PrecisionMismatch"


_TC4_PROBE = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
h = hashlib.sha256()
for (m, n, k, ta, tb, pc) in ((4096, 4096, 1024, False, True, 0), (3000, 2048, 700, False, False, 1),
                              (2048, 1536, 4096, False, True, 1), (4096, 4096, 4096, True, False, 0)):
    A = mp.random_uniform_matrix(k if ta else m, m if ta else k, 11)
    B = mp.random_uniform_matrix(n if tb else k, k if tb else n, 12)
    a = mp.MPArray.from_numpy(A - 0.5, mp.Precision.Half, ctx)
    b = mp.MPArray.from_numpy(B - 0.5, mp.Precision.Half, ctx)
    c = mp.MPArray.from_numpy(np.full((m, n), 0.25), mp.Precision(pc), ctx)
    mp.linalg.gemm(a, b, c, ta, tb, 1.0, -1.0)
    h.update(c.storage().tobytes())
n, nb = 8192, 1024
nt = n // nb
i, j = np.indices((nt, nt))
g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
t.fill_matern(91, 0.5, 0.03, 1.0)
mp.tile_chol(t)
h.update(np.ascontiguousarray(t.to_numpy()).tobytes())
print(h.hexdigest())
"""


def test_gemm_pair_multicast_bitwise():
    """MPCR_TC4=1 (clusters of two CTA pairs sharing A by TMA multicast) only
    changes how operands reach shared memory: dense FP16 GEMMs (even and odd
    N-block counts, ragged M) and an nb = 1024 tiled Cholesky are bit-identical
    to the pair kernel."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(tc4):
        e = dict(os.environ, MPCR_TC4=tc4)
        out = subprocess.run([sys.executable, "-c", _TC4_PROBE, root], env=e, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return out.stdout.strip().splitlines()[-1]

    assert run("1") == run("0")
