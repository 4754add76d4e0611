"""Dense FP64 chol of one 1024 tile (the diagonal-tile POTRF) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
B = rng.random((n, n)); A = B.T @ B + n * np.eye(n)
a = mp.MPArray.from_numpy(A, mp.Precision.Double, ctx)
for _ in range(3):
    u = mp.linalg.chol(a)
ctx.synchronize()
print("ok", u.get(0, 0))
