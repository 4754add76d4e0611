"""GPU parity: precision conversion (bit-exact) and elementwise kernels vs the
reference oracle (oracle/_ref = unmodified mpnum)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, S, D = 0, 1, 2
NP = {H: np.uint16, S: np.float32, D: np.float64}


def special_doubles():
    f16 = np.array([0x0001, 0x03FF, 0x0400, 0x7BFF, 0x3C00, 0x3C01, 0x8001], np.uint16).view(np.float16)
    vals = [0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 65504.0, 65519.99, 65520.0,
            -65520.0, 70000.0, 1 + 2 ** -11, 1 + 3 * 2 ** -12, 2 ** -25, 2 ** -24, 2 ** -24 * 1.5,
            2 ** -14, 2 ** -14 - 2 ** -25, 1e-300, 5e-324, -5e-324, 2.0 ** -149, 2.0 ** -150,
            2.0 ** -126, 3.4028235e38, 3.5e38, -3.5e38, 2047.5, 2048.5, 2049.0, 1e308, 0.1,
            1.0 / 3.0, np.pi]
    vals += list(f16.astype(np.float64))
    # NaN payloads (x86 cvtsd2ss / cvtss2sd keep the top payload bits)
    nan_bits = np.array([0x7FF8000000000001, 0xFFF8000000000000, 0x7FF4000000000000,
                         0x7FFFFFFFFFFFFFFF, 0xFFF0000000000001, 0x7FF8DEADBEEF0000], np.uint64)
    return np.concatenate([np.array(vals, np.float64), nan_bits.view(np.float64)])


def raw_inputs(p, rng):
    if p == H:
        return np.arange(65536, dtype=np.uint32).astype(np.uint16)  # every half pattern
    if p == S:
        sp = special_doubles().astype(np.float32)
        nanf = np.array([0x7FC00001, 0xFFC00000, 0x7FA00000, 0x7F800001, 0xFFFFFFFF],
                        np.uint32).view(np.float32)
        rnd = (rng.standard_normal(200000) * 10.0 ** rng.integers(-8, 8, 200000)).astype(np.float32)
        sub = (rng.random(10000) * 2.0 ** -126).astype(np.float32)
        return np.concatenate([sp, nanf, rnd, sub])
    sp = special_doubles()
    rnd = rng.standard_normal(200000) * 10.0 ** rng.integers(-12, 12, 200000)
    near_half = (rng.random(100000) - 0.5) * 140000.0
    tiny = (rng.random(50000) - 0.5) * 2.0 ** -12
    ties = (np.arange(1, 5001, dtype=np.float64) * 2.0 + 1.0) * 2.0 ** -11  # RNE ties in half
    return np.concatenate([sp, rnd, near_half, tiny, ties])


@pytest.mark.parametrize("pin", [H, S, D])
@pytest.mark.parametrize("pout", [H, S, D])
def test_convert_bit_exact(ctx, ref, rng, pin, pout):
    import paper_2406_02701_b200 as mp

    raw = raw_inputs(pin, rng)
    a = mp.MPArray.from_storage(raw, raw.size, 1, mp.Precision(pin), ctx)
    got = a.converted(mp.Precision(pout)).storage()
    want = ref.convert(pin, pout, raw)
    g = got.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[got.itemsize])
    w = want.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[want.itemsize])
    mism = np.nonzero(g != w)[0]
    assert mism.size == 0, f"{mism.size} mismatches, first idx {mism[:5]} got {g[mism[:5]]} want {w[mism[:5]]}"



def test_convert_strided_and_odd_lengths(ctx, ref, rng):
    import paper_2406_02701_b200 as mp

    for n in (1, 7, 8, 9, 1023, 4097):
        x = rng.standard_normal(n)
        a = mp.MPArray.from_numpy(x, mp.Precision.Double, ctx)
        got = a.converted(mp.Precision.Half).storage()
        assert np.array_equal(got, ref.encode_f16(x))


def test_from_to_doubles_roundtrip(ctx, rng):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    x = rng.standard_normal((37, 19)) * 1000
    for p in (H, S, D):
        a = mp.MPArray.from_numpy(x, mp.Precision(p), ctx)
        np.testing.assert_array_equal(a.to_numpy(), round_to(x, p))


def _pair(rng, shape, pa, pb):
    from oracle.oracle import round_to

    return round_to(rng.standard_normal(shape) * 3, pa), round_to(rng.standard_normal(shape) * 3, pb)


@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_ew_binary_all_pairs(ctx, ref, rng, op):
    import paper_2406_02701_b200 as mp

    for pa in (H, S, D):
        for pb in (H, S, D):
            A, B = _pair(rng, (33, 17), pa, pb)
            B[0, 0] = 0.0  # division by zero follows IEEE
            da = mp.MPArray.from_numpy(A, mp.Precision(pa), ctx)
            db = mp.MPArray.from_numpy(B, mp.Precision(pb), ctx)
            out = mp.ew_binary(mp.BinaryOp(op), da, db)
            assert out.precision() == max(pa, pb)
            got = out.to_numpy()
            want = ref.ew_binary(op, pa, pb, A, B)
            nan = np.isnan(want)
            assert np.array_equal(np.isnan(got), nan)
            np.testing.assert_array_equal(got[~nan], want[~nan])


def test_ew_half_correctly_rounded(ctx, rng):
    """test_array.cpp:163-175: half add/mul == encode_f16(exact)."""
    import paper_2406_02701_b200 as mp

    bits_a = (rng.integers(0, 0x7BFF, 100000)).astype(np.uint16)
    bits_b = (rng.integers(0, 0x7BFF, 100000)).astype(np.uint16)
    ha, hb = bits_a.view(np.float16).astype(np.float64), bits_b.view(np.float16).astype(np.float64)
    da = mp.MPArray.from_storage(bits_a, bits_a.size, 1, mp.Precision.Half, ctx)
    db = mp.MPArray.from_storage(bits_b, bits_b.size, 1, mp.Precision.Half, ctx)
    s = mp.ew_binary(mp.BinaryOp.Add, da, db).storage()
    m = mp.ew_binary(mp.BinaryOp.Mul, da, db).storage()
    np.testing.assert_array_equal(s, (ha + hb).astype(np.float16).view(np.uint16))
    np.testing.assert_array_equal(m, (ha * hb).astype(np.float16).view(np.uint16))


def test_ew_half_2048_plus_1(ctx):
    import paper_2406_02701_b200 as mp

    big = mp.MPArray.from_doubles([2048.0], 1, 1, mp.Precision.Half, ctx)
    one = mp.MPArray.from_doubles([1.0], 1, 1, mp.Precision.Half, ctx)
    assert mp.ew_binary(mp.BinaryOp.Add, big, one).get(0, 0) == 2048.0


@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_ew_scalar(ctx, ref, rng, op):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    for p in (H, S, D):
        A = round_to(rng.standard_normal((40, 9)) * 5, p)
        for s in (0.1, 3.0, -1.7e-3, 1e5):
            da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
            got = mp.ew_scalar(mp.BinaryOp(op), da, s).to_numpy()
            want = ref.ew_scalar(op, p, A, s)
            np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_ew_unary(ctx, ref, rng, op):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    for p in (H, S, D):
        A = round_to(rng.random((50, 7)) * 4 + 0.01, p)
        if op == 3:
            A = -A
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        got = mp.ew_unary(mp.UnaryOp(op), da).to_numpy()
        want = ref.ew_unary(op, p, A)
        if op in (2, 3):  # sqrt / abs: correctly rounded, bit-exact
            np.testing.assert_array_equal(got, want)
        else:  # log / exp: few-ulp in the compute precision, then storage rounding
            u = {H: 2.0 ** -10, S: 2.0 ** -21, D: 2.0 ** -50}[p]
            np.testing.assert_allclose(got, want, rtol=u, atol=0)


@pytest.mark.parametrize("op", [0, 1, 2, 3, 4])
def test_reduce(ctx, ref, rng, op):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    for p in (H, S, D):
        A = round_to(rng.standard_normal((1000, 31)), p)
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        got = mp.reduce(mp.ReduceOp(op), da)
        want = ref.reduce(op, p, A)
        if op in (2, 3):
            assert got == want
        else:
            assert abs(got - want) <= 1e-13 * max(1.0, np.abs(A).sum())


def test_reduce_exact_half_sum(ctx):
    """test_array.cpp:211-214: 1e6 halves of 2^-10 sum exactly."""
    import paper_2406_02701_b200 as mp

    h = mp.MPArray.from_storage(np.full(1000000, np.float16(2 ** -10)).view(np.uint16),
                                1000000, 1, mp.Precision.Half, ctx)
    assert mp.reduce(mp.ReduceOp.Sum, h) == 976.5625


def test_reduce_empty_raises(ctx):
    import paper_2406_02701_b200 as mp

    z = mp.MPArray.zeros_matrix(0, 0, mp.Precision.Double, ctx)
    with pytest.raises(mp.MPError) as e:
        mp.reduce(mp.ReduceOp.Sum, z)
    assert e.value.kind == "EmptyArray"


def test_transpose_diag(ctx, ref, rng):
    import paper_2406_02701_b200 as mp
    from oracle.oracle import round_to

    for p in (H, S, D):
        A = round_to(rng.standard_normal((70, 45)), p)
        da = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        np.testing.assert_array_equal(mp.transpose(da).to_numpy(), A.T)
        np.testing.assert_array_equal(mp.diag(da).to_doubles(), ref.diag(p, A))


def test_get_set_bounds(ctx):
    import paper_2406_02701_b200 as mp

    a = mp.MPArray.zeros_matrix(3, 4, mp.Precision.Single, ctx)
    a.set(2, 3, 1.0 / 3.0)
    assert a.get(2, 3) == float(np.float32(1.0 / 3.0))
    with pytest.raises(mp.MPError) as e:
        a.get(3, 0)
    assert e.value.kind == "IndexOutOfRange"
