"""One eager mixed-precision factorization (n = 65536, nb = 1024, bench map):
used under ncu to capture the INT8-digit GEMM and the digit slicer in situ
(-k regex:"oz_" -s <skip> -c <count>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2406_02701_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nb = 1024
ctx = mp.Context(0)
g = bench.band_map(n // nb, 1, 2)
x, y, _ = bench.grid_points(n)
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A.fill_matern_points(x, y, 0.5, 0.03, 1.0, 0.0)
mp.tile_chol(A)
ctx.synchronize()
print("ok", A.logdet())
