#!/bin/bash
# L2 prefetch of the next unit's first k-blocks in the pair kernel
cd "$(dirname "$0")/.."
o=gpurun_out/r02aq
mkdir -p $o
MPCR_TC_L2PF=8 timeout 900 python -m pytest tests/test_gpu_tile.py -q -x -k "bitwise or oracle" > $o/t.log 2>&1; echo "tile rc=$?"; tail -2 $o/t.log
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4))"; }
for v in 0 8 4 16 0 8; do
  MPCR_TC_L2PF=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "pf=$v rc=$? $(summ $o/bench.json)"
done
