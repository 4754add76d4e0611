"""FP16 tcgen05 GEMM rate per operand layout (NN / NT / TN / TT) at m=n=8192."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_02701_b200 as mp  # noqa: E402

ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
m = n = 8192
for k in (1024, 8192):
    for ta, tb in ((False, False), (False, True), (True, False), (True, True)):
        rng = np.random.default_rng(0)
        a = mp.MPArray.from_numpy(rng.random((k, m) if ta else (m, k)) - 0.5, mp.Precision.Half, ctx)
        b = mp.MPArray.from_numpy(rng.random((n, k) if tb else (k, n)) - 0.5, mp.Precision.Half, ctx)
        c = mp.MPArray.from_numpy(rng.random((m, n)), mp.Precision.Half, ctx)
        for _ in range(3):
            mp.linalg.gemm(a, b, c, ta, tb, -1.0, 1.0)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        for _ in range(reps):
            mp.linalg.gemm(a, b, c, ta, tb, -1.0, 1.0)
        e1.record(st)
        ctx.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"k={k:5d} {'T' if ta else 'N'}{'T' if tb else 'N'} {ms:7.3f} ms {2 * m * n * k / ms / 1e9:7.1f} TF/s")
