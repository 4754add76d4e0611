"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libmpnum_ref.so, built from /root/reference by oracle/Makefile).

Run in the build container (the reference sources are not on the GPU box):
    python tests/golden/make_golden.py
The fixtures are small and committed; tests/test_oracle.py pins the C port
(oracle/mpnum_oracle.c) to them and the GPU tests use them as known answers.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402


def main():
    orc.build()
    ref = orc.Ref()
    out = {}
    # --- casts: test_precision.cpp:97-155 known answers + boundary set ------
    kat_x = np.array([0.0, -0.0, 1.0, 65504.0, 65520.0, -65520.0, 70000.0, 1.0 + 2 ** -11,
                      1.0 + 3 * 2 ** -12, np.nan, np.inf, 2 ** -25, 2 ** -24, 1e-300,
                      65503.999, 65519.999, 65520.001, 2047.5, 2048.5, 2049.0, 2 ** -14,
                      2 ** -14 - 2 ** -25, 2 ** -25 * 1.0000001, 2 ** -24 * 1.5])
    kat_x = np.concatenate([kat_x, -kat_x])
    out["kat_x"] = kat_x
    out["kat_f16"] = ref.encode_f16(kat_x)
    allp = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    out["all_half_decoded"] = ref.decode_f16(allp)
    out["all_half_roundtrip"] = ref.encode_f16(ref.decode_f16(allp))
    rs = ref.rng_uniform(20240817, 60000)
    xs = np.concatenate([(rs[:20000] - 0.5) * 140000.0, (rs[20000:40000] - 0.5) * 4.0,
                         (rs[40000:] - 0.5) * 2.0 ** -12])
    out["rand_x"] = xs
    out["rand_f16"] = ref.encode_f16(xs)
    for pin, name in ((2, "d"), (1, "s"), (0, "h")):
        src = {2: xs, 1: xs.astype(np.float32), 0: ref.encode_f16(xs)}[pin]
        for pout, oname in ((2, "d"), (1, "s"), (0, "h")):
            out[f"cvt_{name}{oname}"] = ref.convert(pin, pout, src)
        out[f"cvt_src_{name}"] = src
    # --- dense kernels on Rng(1000+n) uniform inputs (acceptance.cpp:160) ---
    for p in (0, 1, 2):
        n = 24
        u = ref.rng_uniform(1000 + n, 3 * n * n)
        A = orc.round_to(u[: n * n].reshape((n, n), order="F"), p)
        B = orc.round_to(u[n * n: 2 * n * n].reshape((n, n), order="F"), p)
        Cm = orc.round_to(u[2 * n * n:].reshape((n, n), order="F"), p)
        out[f"gemm_A_{p}"], out[f"gemm_B_{p}"], out[f"gemm_C_{p}"] = A, B, Cm
        for ta in (0, 1):
            for tb in (0, 1):
                out[f"gemm_out_{p}_{ta}{tb}"] = ref.gemm(p, p, p, A, B, Cm, ta, tb, 0.7, 0.3)
        S = ref.crossprod(2, u[: n * n].reshape((n, n), order="F")) + n * np.eye(n)
        S = orc.round_to(S, p)
        out[f"chol_in_{p}"] = S
        U = ref.chol(p, S)
        out[f"chol_out_{p}"] = U
        Bt = orc.round_to(u[n * n: n * n + 5 * n].reshape((n, 5), order="F"), p)
        out[f"trsm_B_{p}"] = Bt
        out[f"trsm_out_{p}"] = ref.trsm(p, p, U, Bt, False, True, True, 1.25)
    # --- MPCRTile: paper 4x4 and a mixed n=128 case ------
    xs4 = np.array([(x, y) for y in (0.0, 1.0) for x in (0.0, 1.0)])
    M = np.exp(-np.sqrt(((xs4[:, None] - xs4[None]) ** 2).sum(-1)))
    out["paper_M"] = M
    out["paper_L"] = ref.tile_chol(4, 2, np.array([[2, 1], [1, 2]]), M)
    n, nb = 128, 32
    cov = ref.grid_matern(12, n, 0.5, 0.1, 1.0, 2)
    g = np.array([[2 if i == j else (1 if abs(i - j) == 1 else 0) for j in range(4)]
                  for i in range(4)])
    out["tile_cov"], out["tile_prec"] = cov, g
    out["tile_L"] = ref.tile_chol(n, nb, g, cov)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
