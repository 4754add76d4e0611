"""Self-checks of a factored MPCRTile that do not need the factor on the host.

At the north-star sizes (n = 65536 / 131072) the factor is 9-35 GB and the
CPU oracle cannot factor the matrix at all, so correctness is checked on a
sample (the reference attaches an error to every timing:
proj/tools/mpnum_cli.cpp:59-63,174 and the chol band of
proj/tests/acceptance.cpp:179-187):

* ``sampled_residual``: rows R of L are downloaded (mp_tile_get_rows) and
  E = (L L^T)[R, R] - A[R, R] is formed in FP64 on the host, with A[R, R]
  recomputed from the point coordinates by the Matern closed form
  (covariance.cpp:58-67) and rounded to each entry's tile precision with
  numpy's correctly rounded casts (the set_linear semantics of
  array.cpp:97-133).  R mixes clusters of consecutive rows (near-diagonal
  entries, where the covariance is large) spread over the whole matrix —
  including the last tile row, which received every trailing update — and
  random rows.
* ``leading_rows_equal``: the tiled right-looking algorithm updates tile
  (i, j) only from panels k < min(i, j), so the leading m x m tiles of the
  factor are the factor of the leading m x m principal submatrix — computed
  by exactly the same per-tile kernels.  The large factor's leading block
  must therefore equal, bit for bit, a separate factorization of the
  leading sub-problem, which is small enough for the CPU oracle.

This module never touches ``oracle/``; the tests and bench.py use it.
"""
from __future__ import annotations

import numpy as np


def grid_points(n: int, side: int | None = None):
    """First n points of a side x side unit grid, x fastest
    (covariance.cpp:9-21); side defaults to ceil(sqrt(n))."""
    if side is None:
        side = max(int(np.ceil(np.sqrt(n))), 2)
    p = np.arange(n)
    return (p % side) / (side - 1), (p // side) / (side - 1), side


def band_map(nt: int, b64: int, b32: int) -> np.ndarray:
    """Tile precision by band |i - j|: < b64 FP64 (2), < b32 FP32 (1), else FP16 (0)."""
    i, j = np.indices((nt, nt))
    d = np.abs(i - j)
    return np.where(d < b64, 2, np.where(d < b32, 1, 0)).astype(np.int32)


def sample_rows(n: int, nb: int, clusters: int = 8, width: int = 16, extra: int = 64,
                seed: int = 0) -> np.ndarray:
    """Sorted unique row indices: `clusters` runs of `width` consecutive rows
    spread over [0, n) (the last run ends at row n - 1) plus `extra` random rows."""
    starts = np.linspace(0, n - width, clusters).astype(np.int64)
    rows = [np.arange(s, s + width) for s in starts]
    rows.append(np.random.default_rng(seed).integers(0, n, extra))
    return np.unique(np.concatenate(rows))


def round_to_grid(v: np.ndarray, prec: np.ndarray) -> np.ndarray:
    """Round doubles to per-entry precisions (0 half, 1 single, 2 double)."""
    with np.errstate(over="ignore"):
        h = v.astype(np.float16).astype(np.float64)
        s = v.astype(np.float32).astype(np.float64)
    return np.where(prec == 0, h, np.where(prec == 1, s, v))


def matern05_block(x, y, ri, ci, range_: float, variance: float = 1.0, nugget: float = 0.0):
    """sigma2 * exp(-d / range) (+ nugget on the diagonal) for rows ri, cols ci."""
    d = np.hypot(x[ri][:, None] - x[ci][None, :], y[ri][:, None] - y[ci][None, :])
    a = variance * np.exp(-d / range_)
    a = a + nugget * (ri[:, None] == ci[None, :])
    return a


def sampled_residual(tile, x, y, rows, nb: int, prec_grid: np.ndarray, range_: float,
                     variance: float = 1.0, nugget: float = 0.0, L_rows: np.ndarray | None = None):
    """Backward error of a factored MPCRTile on the sample R = rows.

    Returns normwise ||E||_F / ||A[R,R]||_F, the largest entry max|E| / max|A|
    and the sample size, E = (L L^T)[R,R] - A[R,R]."""
    rows = np.asarray(rows, dtype=np.int64)
    if L_rows is None:
        L_rows = tile.get_rows(rows)
    A = matern05_block(x, y, rows, rows, range_, variance, nugget)
    A = round_to_grid(A, prec_grid[rows[:, None] // nb, rows[None, :] // nb])
    LLt = L_rows @ L_rows.T
    E = LLt - A
    return {"normwise": float(np.linalg.norm(E) / np.linalg.norm(A)),
            "max_entry": float(np.abs(E).max() / np.abs(A).max()),
            "rows": int(rows.size), "entries": int(rows.size) ** 2}


def leading_rows_equal(L_rows_big: np.ndarray, L_rows_small: np.ndarray) -> bool:
    """Rows of the big factor restricted to the leading m columns vs the same
    rows of the factor of the leading m x m sub-problem: bit for bit."""
    m = L_rows_small.shape[1]
    return bool(np.array_equal(L_rows_big[:, :m], L_rows_small))
