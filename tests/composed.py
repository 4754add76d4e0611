"""TEST INFRASTRUCTURE: the reference's tiled-Cholesky composition run with the
engine's DENSE entry points, as a second, independent implementation of the
mixed-precision algorithm at sizes the CPU oracle cannot reach.

It performs exactly the calls of oracle/ref_shim.cpp:ref_tile_chol (SURVEY
§8c) — per step k: linalg::chol(A_kk) (upper U), A_kk <- U^T;
trsm(U.converted(p_ik), A_ik, Right, upper, no-trans, 1) for i > k;
gemm(A_ik.converted(p_ij), A_jk.converted(p_ij), A_ij, {N, T, -1, 1}) for
j > k, i >= j — but through mp_chol / mp_trsm / mp_gemm / mp_convert on tile
views (each of those is checked per operation against the reference CPU
library in tests/test_gpu_linalg.py).  It shares none of the fused
scheduler's machinery (no lookahead, no inverses, no TRSM-as-GEMM, no INT8
digits, no DMMA widening inside updates): where the two factorizations agree
to within the mixed-precision rounding budget, the fused path is checked.
"""
from __future__ import annotations

import numpy as np


def composed_tile_chol(t, nb: int, g: np.ndarray) -> None:
    """Factor the MPCRTile t in place (lower L in the lower tiles; the upper
    tiles are left as they were)."""
    import paper_2406_02701_b200 as mp
    from paper_2406_02701_b200._lib import check, lib

    ctx = t.ctx
    nt = g.shape[0]
    L = lib()
    view = {}

    def tile(i, j):
        key = (i, j)
        if key not in view:
            view[key] = t.GetTile(i + 1, j + 1)
        return view[key]

    # one reusable conversion buffer per precision and operand slot
    buf = {(p, s): mp.MPArray.zeros_matrix(nb, nb, mp.Precision(p), ctx) for p in range(3) for s in range(2)}

    def as_prec(a, p_from, p_to, slot):
        if p_from == p_to:
            return a
        b = buf[(p_to, slot)]
        check(L.mp_convert(ctx.h, a.h, b.h))
        return b

    for k in range(nt):
        u = mp.linalg.chol(tile(k, k))  # upper; NotPositiveDefinite raises
        check(L.mp_transpose(ctx.h, u.h, tile(k, k).h))
        for i in range(k + 1, nt):
            uc = as_prec(u, int(g[k, k]), int(g[i, k]), 0)
            mp.linalg.trsm(uc, tile(i, k), mp.Side.Right, True, False, 1.0)
        for j in range(k + 1, nt):
            for i in range(j, nt):
                pc = int(g[i, j])
                a = as_prec(tile(i, k), int(g[i, k]), pc, 0)
                b = as_prec(tile(j, k), int(g[j, k]), pc, 1)
                mp.linalg.gemm(a, b, tile(i, j), False, True, -1.0, 1.0)
        u.close()
    ctx.synchronize()
