#!/bin/bash
# INT8-digit tiles with both paired sources take both panels in one pass
cd "$(dirname "$0")/.."
o=gpurun_out/r02w
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "half_to_double or int8 or digit" > $o/t_linalg.log 2>&1; echo "linalg-oz rc=$?"; tail -2 $o/t_linalg.log
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -3 $o/t_tile.log
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --b32 4 > $o/bench_b32_4.json 2> $o/bench_b32_4.err; echo "bench b32=4 rc=$? $(summ $o/bench_b32_4.json)"
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
