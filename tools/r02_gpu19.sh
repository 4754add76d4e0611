#!/bin/bash
# oz: unit counter drawn one unit ahead
cd "$(dirname "$0")/.."
o=gpurun_out/r02q
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "half_to_double or int8 or digit" > $o/t_linalg.log 2>&1; echo "linalg-oz rc=$?"; tail -2 $o/t_linalg.log
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 40 -c 1 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
