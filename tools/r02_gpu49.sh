#!/bin/bash
# knob sweep with paired steps: pair-kernel stages, C evict-first, persistence
cd "$(dirname "$0")/.."
o=gpurun_out/r02au
mkdir -p $o
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4))"; }
for v in "X=1" "MPCR_TC2_STAGES=5" "MPCR_C_EVICT_FIRST=0" "MPCR_TILES_PER_CTA=0" "MPCR_UPDATE_GROUP=32" "X=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "$v rc=$? $(summ $o/bench.json)"
done
