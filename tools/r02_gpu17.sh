#!/bin/bash
# digit-count histogram (per 128-row block) and the b32=4 line
cd "$(dirname "$0")/.."
o=gpurun_out/r02o
mkdir -p $o
MPCR_DEBUG_NDIG=1 timeout 300 python tools/oz_insitu.py 65536 > $o/ndig.txt 2>&1; echo "ndig rc=$?"
python - <<'PY'
import re
h=[0]*8
for l in open('gpurun_out/r02o/ndig.txt'):
    m=re.match(r'\[mpcr\] step (\d+) digits:(.*)',l)
    if m:
        v=list(map(int,m.group(2).split()))
        h=[a+b for a,b in zip(h,v)]
print("block digit histogram (0..7):", h)
PY
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --b32 4 > $o/bench_b32_4.json 2> $o/bench_b32_4.err; echo "bench b32=4 rc=$?"
python -c "import json;d=json.loads(open('$o/bench_b32_4.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], d['accuracy'], {k:(round(v['ms'],1), round(v.get('tflops',0) or 0,1)) for k,v in d['breakdown']['classes'].items()})"
