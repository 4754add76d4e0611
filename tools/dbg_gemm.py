import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
rng = np.random.default_rng(0)
def run(pa, pc, m, n, k, ta, tb):
    A = rng.random((k, m) if ta else (m, k)) - 0.5
    B = rng.random((n, k) if tb else (k, n)) - 0.5
    A = A.astype(np.float16).astype(np.float64) if pa == 0 else A.astype(np.float32).astype(np.float64)
    B = B.astype(np.float16).astype(np.float64) if pa == 0 else B.astype(np.float32).astype(np.float64)
    da = mp.MPArray.from_numpy(A, mp.Precision(pa), ctx); db = mp.MPArray.from_numpy(B, mp.Precision(pa), ctx)
    dc = mp.MPArray.zeros_matrix(m, n, mp.Precision(pc), ctx)
    mp.linalg.gemm(da, db, dc, ta, tb, 1.0, 0.0)
    G = dc.to_numpy(); W = (A.T if ta else A) @ (B.T if tb else B)
    bad = np.abs(G - W) > 1e-3 * np.abs(W).max()
    rows = np.nonzero(bad.any(1))[0]; cols = np.nonzero(bad.any(0))[0]
    print(f"pa{pa} pc{pc} {m}x{n}x{k} ta{int(ta)} tb{int(tb)}: rel {np.linalg.norm(G-W)/np.linalg.norm(W):.2e} bad {bad.sum()} rows[{rows.min() if rows.size else '-'}..{rows.max() if rows.size else '-'}] cols[{cols.min() if cols.size else '-'}..{cols.max() if cols.size else '-'}]", flush=True)
for (m, n, k) in [(256, 256, 64), (256, 300, 64), (200, 256, 64), (256, 256, 136), (200, 300, 136)]:
    for ta in (False, True):
        for tb in (False, True):
            run(0, 1, m, n, k, ta, tb)
for (m, n, k) in [(256, 256, 64), (256, 256, 32), (512, 512, 256)]:
    for ta in (False, True):
        for tb in (False, True):
            run(1, 1, m, n, k, ta, tb)
