#!/bin/bash
# oz epilogue fast path; FP32 tiles on INT8 digits (MPCR_OZAKI32)
cd "$(dirname "$0")/.."
o=gpurun_out/r02r
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x > $o/t_linalg.log 2>&1; echo "linalg rc=$?"; tail -2 $o/t_linalg.log
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -3 $o/t_tile.log
timeout 1200 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > $o/t_nb1024.log 2>&1; echo "nb1024 rc=$?"; tail -2 $o/t_nb1024.log; grep -o "n=.*err.*" $o/t_nb1024.log | cut -c1-150
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --b32 4 > $o/bench_b32_4.json 2> $o/bench_b32_4.err; echo "bench b32=4 rc=$? $(summ $o/bench_b32_4.json)"
MPCR_OZAKI32=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --b32 4 > $o/bench_b32_4_dmma.json 2> $o/bench_b32_4_dmma.err; echo "bench b32=4 dmma rc=$? $(summ $o/bench_b32_4_dmma.json)"
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 40 -c 1 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
