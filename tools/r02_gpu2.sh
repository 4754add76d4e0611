#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 tools/micro/run_peaks.sh gpurun_out/r02_peaks > /dev/null 2>&1; echo "peaks rc=$?"
timeout 1500 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > gpurun_out/r02_t_nb1024.log 2>&1; echo "nb1024 rc=$?"
timeout 1200 python -m pytest tests/test_gpu_tile.py tests/test_gpu_linalg.py -q -x > gpurun_out/r02_t_tile.log 2>&1; echo "tile rc=$?"
tail -3 gpurun_out/r02_t_tile.log
