"""FP16 NT GEMM of the Cholesky update shape (C 8192 x 8192 half, K = 1024)
with beta = 1 (read-modify-write of C, as the trailing update) vs beta = 0
(store only): how much the epilogue's C read costs the pair kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
m = n = 8192
rng = np.random.default_rng(0)
for k in (1024, 4096):
    a = mp.MPArray.from_numpy(rng.random((m, k)) - 0.5, mp.Precision.Half, ctx)
    b = mp.MPArray.from_numpy(rng.random((n, k)) - 0.5, mp.Precision.Half, ctx)
    c = mp.MPArray.from_numpy(rng.random((m, n)), mp.Precision.Half, ctx)
    for beta in (1.0, 0.0):
        for _ in range(3):
            mp.linalg.gemm(a, b, c, False, True, -1.0, beta)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            mp.linalg.gemm(a, b, c, False, True, -1.0, beta)
        e1.record(st)
        ctx.synchronize()
        t = e0.elapsed_time(e1) / 10
        print(f"k={k} beta={beta}: {t * 1e3:8.1f} us  {2 * m * n * k / (t * 1e-3) / 1e12:7.1f} TFLOP/s")
