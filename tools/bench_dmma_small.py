"""Time the small FP64 DMMA GEMMs of the Cholesky critical path (the TRTRI
levels and the FP64 diagonal SYRK with an FP32 panel) through linalg.gemm:
C(m x m, double) += A(m x k) B(m x k)^T for m in {512, 1024}, k = m, with
double and single operands.  Usage: python tools/bench_dmma_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
rng = np.random.default_rng(0)
for m in (512, 1024):
    for prec in (mp.Precision.Double, mp.Precision.Single):
        a = mp.MPArray.from_numpy(rng.random((m, m)) - 0.5, prec, ctx)
        b = mp.MPArray.from_numpy(rng.random((m, m)) - 0.5, prec, ctx)
        c = mp.MPArray.from_numpy(rng.random((m, m)), mp.Precision.Double, ctx)
        for _ in range(3):
            mp.linalg.gemm(a, b, c, False, True, -1.0, 1.0)
        ctx.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            mp.linalg.gemm(a, b, c, False, True, -1.0, 1.0)
            e1.record(st)
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(f"m=n=k={m} {prec.name:6s} operands -> double: {t * 1e3:7.1f} us, "
              f"{2 * m ** 3 / (t * 1e-3) / 1e12:5.1f} TFLOP/s")
