#!/bin/bash
# paired steps: correctness (tile suite, dist simulation, nb=1024 parity) and A/B bench
cd "$(dirname "$0")/.."
o=gpurun_out/r02i
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
for v in 1 0; do
  MPCR_PAIR_STEPS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_pair$v.json 2> $o/bench_pair$v.err; echo "bench pair=$v rc=$?"
  python -c "import json;d=json.loads(open('$o/bench_pair$v.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"
done
