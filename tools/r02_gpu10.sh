#!/bin/bash
cd "$(dirname "$0")/.."
o=gpurun_out/r02h
mkdir -p $o
for v in "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=4" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=8" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=16" "MPCR_CAST_CTAS=2 MPCR_CAST_U=4" "MPCR_CAST_CTAS=8 MPCR_CAST_U=2" "MPCR_CAST_CTAS=4 MPCR_CAST_U=1"; do
  env $v timeout 120 python bench.py --workload cast --cast half:single --n 8192 --steps 500 --warmup 20 --no-cpu > $o/cast_hs.json 2>> $o/err.log
  echo "$v: $(python -c "import json;d=json.loads(open('$o/cast_hs.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['samples'])" 2>&1 | tail -1)"
done
timeout 300 python tools/oz_insitu.py 65536 > $o/oz_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"oz_" -s 40 -c 2 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
