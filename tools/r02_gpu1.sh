#!/bin/bash
# round-2 GPU check: new nb=1024 parity tests, the full GPU suite, default bench
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt
timeout 1500 python -m pytest tests/test_gpu_tile_nb1024.py -x -q -s > gpurun_out/r02_t_nb1024.log 2>&1; echo "nb1024 rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -k "not nb1024" > gpurun_out/r02_t_all.log 2>&1; echo "all rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r02_t_all.log
