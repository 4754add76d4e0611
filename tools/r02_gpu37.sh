#!/bin/bash
# direct head solve, again, now that the next head waits for its own tile only
cd "$(dirname "$0")/.."
o=gpurun_out/r02ai
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py tests/test_gpu_nll.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -15 $o/t_tile.log | grep -E "passed|failed|Error|assert" | head -5
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain.txt 2>&1; echo "chain rc=$?"; tail -2 $o/chain.txt
MPCR_DIRECT_HEAD=0 timeout 600 python tools/chain_time.py 131072 1024 > $o/chain0.txt 2>&1; echo "chain0 rc=$?"; tail -2 $o/chain0.txt
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'])"; }
for v in 1 0 1 0; do
MPCR_DIRECT_HEAD=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench direct=$v rc=$? $(summ $o/bench.json)"
done
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
