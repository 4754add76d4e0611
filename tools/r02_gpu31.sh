#!/bin/bash
# A/B: oz epilogue 8 warps (64 columns) vs 12 warps (48/48/32), same box, alternating
cd "$(dirname "$0")/.."
o=gpurun_out/r02ac
mkdir -p $o
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);c=d['breakdown']['classes'];print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), 'int8', round(c['gemm_f64_int8']['ms'],1), 'f16', round(c['gemm_f16']['ms'],1))"; }
for v in epi8 epi12 epi8 epi12 epi8 epi12; do
  cp tools/ab/lib_$v.so paper_2406_02701_b200/libmpcr_b200.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "$v rc=$? $(summ $o/bench.json)"
done
