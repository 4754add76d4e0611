#!/bin/bash
# paired steps with tile column k+2 on the lookahead stream (4 panel generations)
cd "$(dirname "$0")/.."
o=gpurun_out/r02m
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x > $o/t_linalg.log 2>&1; echo "linalg rc=$?"; tail -2 $o/t_linalg.log
