"""FP16 x FP16 -> FP64 GEMM through the INT8 digit path vs FP64 DMMA."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
for n in (2048, 4096, 8192):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    for pa, label in ((mp.Precision.Half, "int8-digits"), (mp.Precision.Double, "dmma")):
        da = mp.MPArray.from_numpy(A, pa, ctx)
        db = mp.MPArray.from_numpy(B, pa, ctx)
        dc = mp.MPArray.from_numpy(np.zeros((n, n)), mp.Precision.Double, ctx)
        for _ in range(2):
            mp.linalg.gemm(da, db, dc, False, True, -1.0, 1.0)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(st)
        for _ in range(reps):
            mp.linalg.gemm(da, db, dc, False, True, -1.0, 1.0)
        e1.record(st)
        ctx.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"n={n:5d} {label:12s} {ms:8.3f} ms  {2 * n ** 3 / ms / 1e9:8.1f} TFLOP/s (FP64-equivalent)")
