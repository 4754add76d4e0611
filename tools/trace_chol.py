"""Timeline of one tiled Cholesky (per-launch start/end on both streams) and
where the main stream idles.  Usage: python tools/trace_chol.py [n] [nb] [out.csv]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_02701_b200 as mp  # noqa: E402

CLS = ["gemm_f16", "gemm_f32", "gemm_f64", "potrf_trtri", "trsm", "cast", "other", "gemm_f64_int8"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/trace.csv"
ctx = mp.Context(0)
g = bench.band_map(n // nb, 1, 2)
x, y, _ = bench.grid_points(n)
A0 = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
A0.fill_matern_points(x, y, 0.5, 0.03, 1.0, 0.0)
for _ in range(2):
    A.copy_from(A0)
    mp.tile_chol(A)
A.copy_from(A0)
ctx.synchronize()
ctx.prof_enable(True)
ctx.prof_trace(True)
mp.tile_chol(A)
ctx.synchronize()
ctx.prof_trace_dump(out)
ctx.prof_enable(False)
d = np.genfromtxt(out, delimiter=",", names=True)
t0 = d["start_ms"].min()
T = d["end_ms"].max() - t0
print(f"n={n} nb={nb}: chol span {T:.2f} ms, {len(d)} timed launches")
for st in (0, 1, 2):
    m = d["stream"] == st
    if not m.any():
        continue
    busy = (d["end_ms"][m] - d["start_ms"][m]).sum()
    print(f" stream {st}: busy {busy:.2f} ms ({busy / T:.0%})")
    for c in range(len(CLS)):
        mc = m & (d["cls"] == c)
        if mc.any():
            print(f"    {CLS[c]:12s} {(d['end_ms'][mc] - d['start_ms'][mc]).sum():8.2f} ms  {mc.sum():5d} launches")
# idle on the main stream: gaps between consecutive launches
m = d["stream"] == 0
s0 = np.sort(np.stack([d["start_ms"][m], d["end_ms"][m]], 1), axis=0)
iv = s0[np.argsort(s0[:, 0])]
gaps, cur = [], iv[0, 1]
for a, b in iv[1:]:
    if a > cur:
        gaps.append((cur - t0, a - cur))
    cur = max(cur, b)
gaps = np.array(gaps) if gaps else np.zeros((0, 2))
print(f" main-stream idle: {gaps[:, 1].sum():.2f} ms in {len(gaps)} gaps; largest:",
      [(round(a, 1), round(b, 2)) for a, b in sorted(gaps.tolist(), key=lambda z: -z[1])[:8]])
# per-step idle split: first/second half of the factorization
half = T / 2
print(f"   idle in first half {gaps[gaps[:, 0] < half, 1].sum():.2f} ms, second half "
      f"{gaps[gaps[:, 0] >= half, 1].sum():.2f} ms")
