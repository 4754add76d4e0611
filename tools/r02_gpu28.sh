#!/bin/bash
# config lines refreshed at the final code (casts after the per-direction tuning,
# FP16 x FP16 -> FP64 on INT8 digits, NLL at n = 65536 with paired steps)
cd "$(dirname "$0")/.."
o=gpurun_out/r02z
mkdir -p $o
B="python bench.py"
for d in half:single single:half half:double double:half single:double double:single; do
  timeout 300 $B --workload cast --cast $d --n 8192 --steps 200 --warmup 10 > $o/cast_${d/:/_}_8192.json 2>> $o/err.log; echo "cast $d rc=$?"
done
timeout 600 $B --workload gemm --prec half --cprec double --n 8192 --steps 5 --warmup 3 > $o/gemm_half_double_8192.json 2>> $o/err.log; echo "gemm h->d rc=$?"
timeout 600 $B --workload gemm --prec half --n 8192 --steps 10 --warmup 3 > $o/gemm_half_8192.json 2>> $o/err.log; echo "gemm h rc=$?"
timeout 300 $B --workload gemm --prec single --n 2048 --steps 10 --warmup 3 > $o/gemm_single_2048.json 2>> $o/err.log; echo "g1 rc=$?"
timeout 1200 $B --workload nll --n 65536 --steps 3 --warmup 3 > $o/nll_65536.json 2>> $o/err.log; echo "nll rc=$?"
for f in $o/*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f'.split('/')[-1], round(d['value'],1), d['unit'], (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'], (d.get('e2e') or {}).get('value'))"; done
