#!/bin/bash
# b32 = 4 line at HEAD (FP32 band on INT8 digits vs DMMA)
cd "$(dirname "$0")/.."
o=gpurun_out/r02av
mkdir -p $o
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --b32 4 > $o/b32_4.json 2> $o/b32_4.err; echo "oz32 rc=$?"
MPCR_OZAKI32=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --b32 4 > $o/b32_4_dmma.json 2> $o/b32_4_dmma.err; echo "dmma rc=$?"
for f in $o/b32_4.json $o/b32_4_dmma.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f'.split('/')[-1], round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), 'e2e', round(d['e2e']['value'],1), 'blend', round(d['blended_roofline']['frac'],3), d['accuracy']['sampled_backward_error'])"; done
