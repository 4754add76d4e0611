"""Time the FP64 POTRF of one diagonal tile (n x n, default 1024) as the
tile Cholesky runs it (single-tile MPCRTile: POTRF only, graph replay), plus
the dense chol for ncu.  MPCR_POTRF_TRACE=1 prints the per-phase clocks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
B = rng.random((n, n))
A = B.T @ B + n * np.eye(n)
A0 = mp.MPCRTile(n, n, n, n, A, [[2]], ctx)
T = mp.MPCRTile(n, n, n, n, None, [[2]], ctx)
st = torch.cuda.ExternalStream(ctx.stream())
for _ in range(3):
    T.copy_from(A0)
    mp.tile_chol(T)
ctx.synchronize()
if not os.environ.get("MPCR_POTRF_TRACE"):
    ts = []
    for _ in range(20):
        T.copy_from(A0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        mp.tile_chol(T)
        e1.record(st)
        ctx.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"potrf n={n}: median {np.median(ts) * 1e3:.1f} us, min {min(ts) * 1e3:.1f} us")
L = T.to_numpy()
print("max |L L^T - A| / |A|:", np.abs(L @ L.T - A).max() / np.abs(A).max())
