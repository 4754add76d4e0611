#!/bin/bash
# hybrid bulk launch: multicast clusters of 4 + plain pairs on a side stream
cd "$(dirname "$0")/.."
o=gpurun_out/r02ao
mkdir -p $o
MPCR_TC_HYBRID=1 timeout 900 python -m pytest tests/test_gpu_tile.py -q -x > $o/t_tile.log 2>&1; echo "tile(hybrid) rc=$?"; tail -2 $o/t_tile.log
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'])"; }
for v in "MPCR_TC_HYBRID=0" "MPCR_TC_HYBRID=1" "MPCR_TC_HYBRID=1 MPCR_TC_HYBRID_FRAC=0.85" "MPCR_TC_HYBRID=0" "MPCR_TC_HYBRID=1" "MPCR_TC_HYBRID=1 MPCR_TC_HYBRID_FRAC=0.95"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "$v rc=$? $(summ $o/bench.json)"
done
