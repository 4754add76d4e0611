"""Critical-chain length of the tiled Cholesky: one factorization with the bulk
trailing update skipped (MPCR_CHAIN_ONLY=1, set by this script; the factor is
meaningless) on a diagonally dominant matrix, timed with CUDA events, plus
the per-class event breakdown of the same eager run.  The chain per step is
what bounds a P x Q run once the bulk is divided by P Q.
Usage: python tools/chain_time.py [n] [nb]"""
import os
import sys

os.environ["MPCR_CHAIN_ONLY"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_02701_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nt = n // nb
ctx = mp.Context(0)
g = bench.band_map(nt, 1, 2)
x, y, _ = bench.grid_points(n)
A0 = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A0.fill_matern_points(x, y, 0.5, 0.03, 1.0, 4.0)  # nugget: stays SPD without the bulk
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
st = torch.cuda.ExternalStream(ctx.stream())
ts = []
for it in range(4):
    A.copy_from(A0)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    mp.tile_chol(A)
    e1.record(st)
    ctx.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts[1:]))
A.copy_from(A0)
ctx.synchronize()
ctx.prof_reset()
ctx.prof_enable(True)
mp.tile_chol(A)
ctx.synchronize()
ctx.prof_enable(False)
cls = {}
for c, nm in enumerate(["gemm_f16", "gemm_f32", "gemm_f64", "potrf_trtri", "trsm", "cast", "other", "gemm_f64_int8"]):
    t, cnt, w = ctx.prof_query(c)
    if cnt:
        cls[nm] = (round(t / nt * 1e3, 1), cnt)
print(f"n={n} nb={nb}: chain-only factorization {ms:.2f} ms = {ms / nt * 1e3:.0f} us per step "
      f"(graph replay; steps {nt}); per-step class time us (eager, overlapping): {cls}")
