#!/bin/bash
# next head tile / diagonal tile updated first on the lookahead stream (parts 4, 5)
cd "$(dirname "$0")/.."
o=gpurun_out/r02ah
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py tests/test_gpu_nll.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain.txt 2>&1; echo "chain rc=$?"; tail -2 $o/chain.txt
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'])"; }
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
done
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
