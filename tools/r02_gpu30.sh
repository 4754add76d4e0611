#!/bin/bash
# oz epilogue with 12 warps (48/48/32 columns)
cd "$(dirname "$0")/.."
o=gpurun_out/r02ab
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "half_to_double or int8 or digit" > $o/t_linalg.log 2>&1; echo "linalg rc=$?"; tail -2 $o/t_linalg.log
timeout 900 python -m pytest tests/test_gpu_tile.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
summ() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), d['accuracy']['sampled_backward_error'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$? $(summ $o/bench.json)"
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 64 -c 2 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
