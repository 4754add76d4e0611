"""Break a Gaussian log-likelihood evaluation into fill / chol / full nll."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_02701_b200 as mp  # noqa: E402

n, nb = 65536, 1024
ctx = mp.Context(0)
g = bench.band_map(n // nb, 1, 2)
x, y, _ = bench.grid_points(n)
z = np.random.default_rng(5).standard_normal(n)
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)


def t(f, reps=3):
    f()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ctx.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


fill = lambda: A.fill_matern_points(x, y, 0.5, 0.03, 1.0, 0.0)
print("fill            %.2f ms" % t(fill))
print("fill+chol       %.2f ms" % t(lambda: (fill(), mp.tile_chol(A))))
print("fill+nll(j=0)   %.2f ms" % t(lambda: (fill(), mp.gaussian_nll(z, A, jitter=0.0))))
print("fill+nll(j=1e-6) %.2f ms" % t(lambda: (fill(), mp.gaussian_nll(z, A, jitter=1e-6))))
