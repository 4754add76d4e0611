#!/bin/bash
# POTRF: panel-block TRSM and CTA 0's SYRK on DMMA
cd "$(dirname "$0")/.."
o=gpurun_out/r02ae
mkdir -p $o
timeout 300 python tools/prof_potrf.py 1024 > $o/potrf_time.txt 2>&1; echo "potrf rc=$?"; tail -2 $o/potrf_time.txt
MPCR_POTRF_TRACE=1 timeout 300 python tools/prof_potrf.py 1024 2>&1 | grep "potrf trace" | tail -1
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "chol or solve or trsm or potrf" > $o/t_linalg.log 2>&1; echo "linalg rc=$?"; tail -2 $o/t_linalg.log
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py tests/test_gpu_nll.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain.txt 2>&1; echo "chain rc=$?"; tail -2 $o/chain.txt
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'])"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
