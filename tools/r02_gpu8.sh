#!/bin/bash
cd "$(dirname "$0")/.."
o=gpurun_out/r02f
mkdir -p $o
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
MPCR_OZAKI=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench_nooz.json 2> $o/bench_nooz.err; echo "bench nooz rc=$?"
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
for v in "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=4" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=8" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=16" "MPCR_CAST_CTAS=2 MPCR_CAST_U=4" "MPCR_CAST_CTAS=8 MPCR_CAST_U=2" "MPCR_CAST_CTAS=4 MPCR_CAST_U=1"; do
  env $v timeout 300 python bench.py --workload cast --cast half:single --n 8192 --steps 2000 --warmup 20 --no-cpu > $o/cast_hs.json 2>> $o/err.log
  echo "$v: $(python -c "import json;d=json.loads(open('$o/cast_hs.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])")"
done
