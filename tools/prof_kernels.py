"""One launch of each kernel family the north star asks ncu evidence for, after
a warm-up: casts (6 directions, 8192^2), FP64 DMMA GEMM, FP16 x FP16 -> FP64
INT8-digit GEMM, FP16 tcgen05 GEMM (8192^3), the batched Matern tile
generator (n = 16384, nb = 1024).  Run under ncu with -k filters
(tools/r02_gpu7.sh); plain, it prints the CUDA-event time of each.
Usage: python tools/prof_kernels.py [casts|dmma|ozaki|f16|matern|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_02701_b200 as mp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())


def timed(name, fn, warm=2):
    for _ in range(warm):
        fn()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    ctx.synchronize()
    print(f"{name}: {e0.elapsed_time(e1):.3f} ms", flush=True)


n = 8192
if which in ("casts", "all"):
    for d in ("half:single", "single:half", "half:double", "double:half", "single:double", "double:single"):
        pi, po = (mp.parse_precision(x) for x in d.split(":"))
        a = mp.MPArray.from_numpy(mp.random_uniform_matrix(n, n, 1000 + n), pi, ctx)
        b = mp.MPArray.zeros_matrix(n, n, po, ctx)
        timed(f"cast {d}", lambda: mp.lib().mp_convert(ctx.h, a.h, b.h))
        a.close()
        b.close()
if which in ("dmma", "ozaki", "f16", "all"):
    A = mp.random_uniform_matrix(n, n, 1000 + n)
    B = mp.random_uniform_matrix(n, n, 1000 + n, skip=n * n)
    for tag, p, pc in (("dmma", 2, 2), ("ozaki", 0, 2), ("f16", 0, 0)):
        if which not in (tag, "all"):
            continue
        a = mp.MPArray.from_numpy(A, mp.Precision(p), ctx)
        b = mp.MPArray.from_numpy(B, mp.Precision(p), ctx)
        c = mp.MPArray.zeros_matrix(n, n, mp.Precision(pc), ctx)
        timed(f"gemm {tag}", lambda: mp.linalg.gemm(a, b, c))
if which in ("matern", "all"):
    m, nb = 16384, 1024
    nt = m // nb
    i, j = np.indices((nt, nt))
    g = np.where(i == j, 2, np.where(abs(i - j) == 1, 1, 0))
    t = mp.MPCRTile(m, m, nb, nb, None, g, ctx)
    x = (np.arange(m) % 128) / 127.0
    y = (np.arange(m) // 128) / 127.0
    timed("matern tiles", lambda: t.fill_matern_points(x, y, 0.5, 0.03, 1.0, 0.0))
