"""CPU: the oracle is pinned before it is trusted.

* the C port (oracle/mpnum_oracle.c) reproduces the committed golden vectors
  bit-for-bit (tests/golden/golden.npz, made from the unmodified reference by
  tests/golden/make_golden.py);
* when the reference was compiled here (oracle/_ref), it reproduces the same
  fixtures and agrees with the port on fresh random instances;
* the reference's own known-answer tests (test_precision.cpp, test_linalg.cpp,
  PAPER.md MPCRTile printouts) hold on the port.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def bits(a):
    a = np.asarray(a)
    return a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.itemsize])


def test_f16_known_answers(port):
    """test_precision.cpp:97-112."""
    kat = [(0.0, 0x0000), (-0.0, 0x8000), (1.0, 0x3C00), (65504.0, 0x7BFF), (65520.0, 0x7C00),
           (-65520.0, 0xFC00), (70000.0, 0x7C00), (1.0 + 2 ** -11, 0x3C00),
           (1.0 + 3 * 2 ** -12, 0x3C01), (np.inf, 0x7C00), (2 ** -25, 0x0000),
           (2 ** -24, 0x0001), (1e-300, 0x0000)]
    x = np.array([k for k, _ in kat])
    np.testing.assert_array_equal(port.encode_f16(x), np.array([v for _, v in kat], np.uint16))
    assert port.encode_f16(np.array([np.nan]))[0] == 0x7E00


def test_port_f16_matches_golden(port, gold):
    np.testing.assert_array_equal(port.encode_f16(gold["kat_x"]), gold["kat_f16"])
    np.testing.assert_array_equal(port.encode_f16(gold["rand_x"]), gold["rand_f16"])
    dec = port.decode_f16(np.arange(65536, dtype=np.uint32).astype(np.uint16))
    np.testing.assert_array_equal(bits(dec)[~np.isnan(dec)],
                                  bits(gold["all_half_decoded"])[~np.isnan(dec)])
    assert np.array_equal(np.isnan(dec), np.isnan(gold["all_half_decoded"]))
    np.testing.assert_array_equal(port.encode_f16(dec), gold["all_half_roundtrip"])


def test_f16_roundtrip_all_patterns(port):
    """test_precision.cpp:114-124 / acceptance criterion 1."""
    pats = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    rt = port.encode_f16(port.decode_f16(pats))
    nan = ((pats >> 10) & 0x1F == 0x1F) & (pats & 0x3FF != 0)
    np.testing.assert_array_equal(rt[~nan], pats[~nan])
    assert np.all(rt[nan] == 0x7E00)


def test_numpy_half_cast_is_encode_f16(port, gold):
    """oracle.round_to relies on numpy's f64->f16 cast being encode_f16."""
    x = gold["rand_x"]
    np.testing.assert_array_equal(x.astype(np.float16).view(np.uint16), gold["rand_f16"])


@pytest.mark.parametrize("pin,name", [(2, "d"), (1, "s"), (0, "h")])
def test_port_convert_matches_golden(port, gold, pin, name):
    src = gold[f"cvt_src_{name}"]
    for pout, oname in ((2, "d"), (1, "s"), (0, "h")):
        got = port.convert(pin, pout, src)
        np.testing.assert_array_equal(bits(got), bits(gold[f"cvt_{name}{oname}"]))


@pytest.mark.parametrize("p", [0, 1, 2])
def test_port_dense_matches_golden(port, gold, p):
    A, B, Cm = gold[f"gemm_A_{p}"], gold[f"gemm_B_{p}"], gold[f"gemm_C_{p}"]
    for ta in (0, 1):
        for tb in (0, 1):
            got = port.gemm(p, p, p, A, B, Cm, ta, tb, 0.7, 0.3)
            np.testing.assert_array_equal(bits(got), bits(gold[f"gemm_out_{p}_{ta}{tb}"]))
    U = port.chol(p, gold[f"chol_in_{p}"])
    np.testing.assert_array_equal(bits(U), bits(gold[f"chol_out_{p}"]))
    X = port.trsm(p, p, U, gold[f"trsm_B_{p}"], False, True, True, 1.25)
    np.testing.assert_array_equal(bits(X), bits(gold[f"trsm_out_{p}"]))


def test_port_tile_chol_matches_golden(port, gold):
    L = port.tile_chol(4, 2, np.array([[2, 1], [1, 2]]), gold["paper_M"])
    np.testing.assert_array_equal(bits(L), bits(gold["paper_L"]))
    L = port.tile_chol(128, 32, gold["tile_prec"], gold["tile_cov"])
    np.testing.assert_array_equal(bits(L), bits(gold["tile_L"]))


def test_paper_printout(port, gold):
    """the MPCRTile chol printout, FP32 signature included."""
    L = port.tile_chol(4, 2, np.array([[2, 1], [1, 2]]), gold["paper_M"])
    printed = np.array([[1, 0, 0, 0], [0.3678794, 0.9298735, 0, 0],
                        [0.3678795, 0.1159098, 0.9226211, 0],
                        [0.2431167, 0.2994405, 0.2641753, 0.8839915]])
    np.testing.assert_allclose(L, printed, atol=5.1e-8)


def test_port_chol_errors(port):
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as e:
        port.chol(2, np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.status == 5 and e.value.info == 1


def test_reference_reproduces_golden(ref, gold):
    """The fixtures are reproducible from the reference itself."""
    np.testing.assert_array_equal(ref.encode_f16(gold["rand_x"]), gold["rand_f16"])
    for p in (0, 1, 2):
        got = ref.gemm(p, p, p, gold[f"gemm_A_{p}"], gold[f"gemm_B_{p}"], gold[f"gemm_C_{p}"],
                       1, 0, 0.7, 0.3)
        np.testing.assert_array_equal(bits(got), bits(gold[f"gemm_out_{p}_10"]))
    L = ref.tile_chol(128, 32, gold["tile_prec"], gold["tile_cov"])
    np.testing.assert_array_equal(bits(L), bits(gold["tile_L"]))


def test_port_equals_reference_random(ref, port):
    rng = np.random.default_rng(99)
    from oracle.oracle import round_to

    for _ in range(30):
        m, n, k = (int(v) for v in rng.integers(1, 12, 3))
        p = int(rng.integers(0, 3))
        ta, tb = int(rng.integers(0, 2)), int(rng.integers(0, 2))
        A = round_to(rng.standard_normal((k, m) if ta else (m, k)), p)
        B = round_to(rng.standard_normal((n, k) if tb else (k, n)), p)
        Cm = round_to(rng.standard_normal((m, n)), p)
        a = ref.gemm(p, p, p, A, B, Cm, ta, tb, 1.3, -0.2)
        b = port.gemm(p, p, p, A, B, Cm, ta, tb, 1.3, -0.2)
        np.testing.assert_array_equal(bits(a), bits(b))
    for op in range(4):
        for pa in range(3):
            for pb in range(3):
                A = round_to(rng.standard_normal((5, 4)), pa)
                B = round_to(rng.standard_normal((5, 4)), pb)
                w = ref.ew_binary(op, pa, pb, A, B)
                g = port.ew_binary(op, pa, pb, A, B)
                np.testing.assert_array_equal(np.isnan(w), np.isnan(g))
                np.testing.assert_array_equal(w[~np.isnan(w)], g[~np.isnan(g)])
        for p in range(3):
            A = round_to(rng.standard_normal((6, 3)), p)
            np.testing.assert_array_equal(ref.ew_scalar(op, p, A, 0.3), port.ew_scalar(op, p, A, 0.3))
    for op in range(5):
        A = rng.standard_normal((50, 3))
        assert ref.reduce(op, 2, A) == port.reduce(op, 2, A)
    for s in (3, 77, 1000):
        np.testing.assert_array_equal(ref.rng_uniform(s, 100), port.rng_uniform(s, 100))


def test_tile_oracle_port_equals_reference_mixed(ref, port):
    rng = np.random.default_rng(5)
    n, nb = 96, 24
    cov = ref.grid_matern(10, n, 0.5, 0.2, 1.0, 2)
    for _ in range(3):
        g = rng.integers(0, 3, (4, 4))
        g = np.maximum(g, g.T)
        np.fill_diagonal(g, 2)
        np.testing.assert_array_equal(bits(ref.tile_chol(n, nb, g, cov)),
                                      bits(port.tile_chol(n, nb, g, cov)))


def test_product_rng_matches_reference_stream(ref):
    """mp_rng_uniform / mp_rng_normal (csrc/rng.cpp) reproduce the reference
    Rng (rng.cpp:9-53) bit for bit: the synthetic bench inputs are the
    reference's own streams (acceptance.cpp:158-162, workloads.cpp:41-49)."""
    import paper_2406_02701_b200 as mp

    for seed in (0, 4, 1000 + 2048, 2**63 + 5):
        u = mp.rng_uniform(seed, 4097)
        np.testing.assert_array_equal(u, ref.rng_uniform(seed, 4097))
        np.testing.assert_array_equal(mp.rng_uniform(seed, 100, skip=3997), u[3997:])
        np.testing.assert_array_equal(mp.rng_normal(seed, 1001), ref.rng_normal(seed, 1001))
