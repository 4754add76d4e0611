#!/bin/bash
# warp-uniform Ozaki MMA issuer: correctness, in-situ timing, ncu capture
cd "$(dirname "$0")/.."
o=gpurun_out/r02j
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_tile.py -q -x > $o/t_linalg.log 2>&1; echo "linalg rc=$?"; tail -2 $o/t_linalg.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"
timeout 300 python tools/oz_insitu.py 65536 > $o/oz_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 20 -c 2 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
