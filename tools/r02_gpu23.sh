#!/bin/bash
# bulk CTA retirement interval with paired steps
cd "$(dirname "$0")/.."
o=gpurun_out/r02u
mkdir -p $o
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4))"; }
for v in "MPCR_TILES_PER_CTA=24" "MPCR_TILES_PER_CTA=12" "MPCR_TILES_PER_CTA=16" "MPCR_TILES_PER_CTA=32" "MPCR_TILES_PER_CTA=24"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "bench $v rc=$? $(summ $o/bench.json)"
done
