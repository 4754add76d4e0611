#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 tools/micro/run_peaks.sh gpurun_out/r02_peaks > /dev/null 2>&1; echo "peaks rc=$?"
timeout 1500 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > gpurun_out/r02_t_nb1024.log 2>&1; echo "nb1024 rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x -k "not nb1024" > gpurun_out/r02_t_all.log 2>&1; echo "all rc=$?"
tail -3 gpurun_out/r02_t_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --b32 4 --no-cpu > gpurun_out/r02_bench_b32_4.json 2> gpurun_out/r02_bench_b32_4.err; echo "bench b32=4 rc=$?"
