#!/bin/bash
# multicast pair kernel A/B, dist simulation tests, chain timing
cd "$(dirname "$0")/.."
o=gpurun_out/r02d
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "multicast" > $o/t_tc4.log 2>&1; echo "tc4 test rc=$?"; tail -2 $o/t_tc4.log
timeout 900 python -m pytest tests/test_gpu_dist_sim.py -q -x > $o/t_dist_sim.log 2>&1; echo "dist sim rc=$?"; tail -2 $o/t_dist_sim.log
for v in 0 1; do
  MPCR_TC4=$v MPCR_DEBUG_TC=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_tc4_$v.json 2> $o/bench_tc4_$v.err; echo "bench tc4=$v rc=$?"
  grep "resident" $o/bench_tc4_$v.err | head -2
done
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain_131072.txt 2>&1; echo "chain rc=$?"; tail -2 $o/chain_131072.txt
