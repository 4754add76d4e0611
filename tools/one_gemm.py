"""One FP16 NT GEMM C(8192x8192, half) -= A B^T with K=1024 (the Cholesky
update shape), for ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
m = n = 8192
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
a = mp.MPArray.from_numpy(rng.random((m, k)) - 0.5, mp.Precision.Half, ctx)
b = mp.MPArray.from_numpy(rng.random((n, k)) - 0.5, mp.Precision.Half, ctx)
c = mp.MPArray.from_numpy(rng.random((m, n)), mp.Precision.Half, ctx)
for _ in range(3):
    mp.linalg.gemm(a, b, c, False, True, -1.0, 1.0)
ctx.synchronize()
print("ok")
