#!/bin/bash
cd "$(dirname "$0")/.."
o=gpurun_out/r02g
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_linalg.py -q -x -k "knobs or int8 or large_k or half_to_double" > $o/t.log 2>&1; echo "tests rc=$?"; tail -2 $o/t.log
for v in 16 32; do
  MPCR_OZ_SLICE_ROWS=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench_$v.json 2> $o/bench_$v.err; echo "bench rows=$v rc=$?"
  python -c "import json;d=json.loads(open('$o/bench_$v.json').read().strip().splitlines()[-1]);print(round(d['value'],1), {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"
done
for v in "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=4" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=8" "MPCR_CAST_WIDEN_SMEM=1 MPCR_CAST_WIDEN_CTAS=16" "MPCR_CAST_CTAS=2 MPCR_CAST_U=4" "MPCR_CAST_CTAS=8 MPCR_CAST_U=2" "MPCR_CAST_CTAS=4 MPCR_CAST_U=1"; do
  env $v timeout 200 python bench.py --workload cast --cast half:single --n 8192 --steps 500 --warmup 20 --no-cpu > $o/cast_hs.json 2>> $o/err.log
  echo "$v: $(python -c "import json;d=json.loads(open('$o/cast_hs.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
