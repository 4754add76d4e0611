"""Probe: GPU tiled chol vs composed reference oracle on the leading n x n
block of the 256x256-grid covariance (the block the n=65536 bench factors
first)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_02701_b200 as mp
from oracle.oracle import Ref, OracleError

def band(nt, b64, b32):
    i, j = np.indices((nt, nt)); dd = abs(i - j)
    return np.where(dd < b64, 2, np.where(dd < b32, 1, 0))

ctx = mp.Context(0)
r = Ref(); r.set_num_threads(os.cpu_count())
n, nb, side = int(sys.argv[1]), int(sys.argv[2]), 256
p = np.arange(n); x = (p % side) / (side - 1); y = (p // side) / (side - 1)
d = np.hypot(x[:, None] - x[None], y[:, None] - y[None])
for rng_, b64, b32 in [(0.1, 1, 2), (0.1, 1, 3), (0.03, 1, 2)]:
    g = band(n // nb, b64, b32)
    cov = np.exp(-d / rng_)
    t = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    t.fill_matern_points(x, y, 0.5, rng_, 1.0, 0.0)
    try:
        mp.tile_chol(t); L = t.to_numpy(); gres = "ok"
    except mp.MPError as e:
        L = None; gres = f"FAIL {e.info}"
    try:
        Lr = r.tile_chol(n, nb, g, cov); rres = "ok"
    except OracleError as e:
        Lr = None; rres = f"FAIL {e.info}"
    Ld = np.linalg.cholesky(cov)
    msg = f"range {rng_} b64 {b64} b32 {b32}: gpu {gres} ref {rres}"
    if L is not None and Lr is not None:
        msg += f" |gpu-ref|/|ref| {np.linalg.norm(L-Lr)/np.linalg.norm(Lr):.2e} |ref-fp64| {np.linalg.norm(Lr-Ld)/np.linalg.norm(Ld):.2e} |gpu-fp64| {np.linalg.norm(L-Ld)/np.linalg.norm(Ld):.2e}"
    print(msg, flush=True)
