"""Which covariance settings factor at n=65536 in mixed precision?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_02701_b200 as mp
n, nb, side = 65536, 1024, 256
ctx = mp.Context(0)
p = np.arange(n); x = (p % side) / (side - 1); y = (p // side) / (side - 1)
def band(nt, b64, b32):
    i, j = np.indices((nt, nt)); dd = abs(i - j)
    return np.where(dd < b64, 2, np.where(dd < b32, 1, 0))
for rng_, nug, b32 in [(0.03, 0.0, 2), (0.1, 1e-3, 2), (0.1, 1e-2, 2), (0.03, 1e-4, 2), (0.1, 1e-3, 3), (0.1, 1e-1, 2)]:
    t = mp.MPCRTile(n, n, nb, nb, None, band(n // nb, 1, b32), ctx)
    t.fill_matern_points(x, y, 0.5, rng_, 1.0, nug)
    ctx.synchronize(); t0 = time.time()
    try:
        mp.tile_chol(t); res = f"ok logdet {t.logdet():.6f}"
    except mp.MPError as e:
        res = f"FAIL col {e.info}"
    print(f"range {rng_} nugget {nug} b32 {b32}: {res} ({time.time()-t0:.2f}s)", flush=True)
    t.close()
