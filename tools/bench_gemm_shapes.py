"""FP16 tcgen05 GEMM rate vs K (m = n fixed): is short K (the Cholesky's 1024)
bound by per-tile prologue/epilogue?  Usage: python tools/bench_gemm_shapes.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
m = n = 8192
for k in (512, 1024, 2048, 4096, 8192):
    for beta, pc in ((0.0, mp.Precision.Half), (1.0, mp.Precision.Half), (1.0, mp.Precision.Single)):
        rng = np.random.default_rng(0)
        a = mp.MPArray.from_numpy(rng.random((m, k)) - 0.5, mp.Precision.Half, ctx)
        b = mp.MPArray.from_numpy(rng.random((n, k)) - 0.5, mp.Precision.Half, ctx)
        c = mp.MPArray.from_numpy(rng.random((m, n)), pc, ctx)
        for _ in range(3):
            mp.linalg.gemm(a, b, c, False, True, -1.0, beta)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        for _ in range(reps):
            mp.linalg.gemm(a, b, c, False, True, -1.0, beta)
        e1.record(st)
        ctx.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"k={k:5d} beta={beta} C={pc.name:6s} {ms:7.3f} ms {2 * m * n * k / ms / 1e9:7.1f} TF/s")
