"""Cast kernel sweep (run on a B200): GB/s per direction and size for the
knobs in csrc/cast.cu (MPCR_CAST_CTAS / _U / _WIDEN_SMEM / _WIDEN_CTAS are
read once per process, so each setting runs in its own process)."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_2406_02701_b200 as mp
ctx = mp.Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
res = {}
for n in (8192, 32768):
    for d in ("half:single", "single:half", "half:double", "double:half", "single:double", "double:single"):
        pi, po = (mp.parse_precision(x) for x in d.split(":"))
        a = mp.MPArray.zeros_matrix(n, n, pi, ctx); b = mp.MPArray.zeros_matrix(n, n, po, ctx)
        for _ in range(3): mp.lib().mp_convert(ctx.h, a.h, b.h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20): mp.lib().mp_convert(ctx.h, a.h, b.h)
        e1.record(st); ctx.synchronize()
        ms = e0.elapsed_time(e1) / 20
        es = {0: 2, 1: 4, 2: 8}
        res[f"{d}@{n}"] = n * n * (es[int(pi)] + es[int(po)]) / ms / 1e6
        a.close(); b.close()
print(json.dumps(res))
'''
settings = [dict(MPCR_CAST_CTAS=str(c), MPCR_CAST_U=str(u), MPCR_CAST_WIDEN_CTAS=str(w))
            for c, u, w in itertools.product((2, 4, 8, 16), (1, 2, 4), (4,))]
settings += [dict(MPCR_CAST_WIDEN_SMEM="1", MPCR_CAST_WIDEN_CTAS=str(w)) for w in (2, 8, 16)]
settings += [dict(MPCR_CAST_WIDEN_SMEM="0", MPCR_CAST_CTAS=str(c), MPCR_CAST_U=str(u)) for c in (4, 8) for u in (1, 2)]
out = []
for st in settings:
    env = dict(os.environ, **st)
    r = subprocess.run([sys.executable, "-c", PROBE, ROOT], env=env, capture_output=True, text=True, timeout=600)
    line = {"setting": st, "gbs": json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]}
    print(json.dumps(line), flush=True)
    out.append(line)
