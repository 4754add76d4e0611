#!/bin/bash
# bulk conversions / digit slicing on a side stream
cd "$(dirname "$0")/.."
o=gpurun_out/r02v
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4))"; }
for v in "MPCR_CONVERT_SIDE=1" "MPCR_CONVERT_SIDE=0" "MPCR_CONVERT_SIDE=1" "MPCR_CONVERT_SIDE=0"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "bench $v rc=$? $(summ $o/bench.json)"
done
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
