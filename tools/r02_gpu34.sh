#!/bin/bash
# update-group width with paired steps
cd "$(dirname "$0")/.."
o=gpurun_out/r02af
mkdir -p $o
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4))"; }
for v in 8 4 6 12 16 8; do
  MPCR_UPDATE_GROUP=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "group=$v rc=$? $(summ $o/bench.json)"
done
