#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_cpp_boundary.py tests/test_gpu_linalg.py -q -x -k "facade or dispatch or large_k" -s > gpurun_out/r02_t_api.log 2>&1; echo "api rc=$?"
tail -3 gpurun_out/r02_t_api.log
timeout 1800 python -m pytest tests/test_gpu_tile_nb1024.py -q -s > gpurun_out/r02_t_nb1024.log 2>&1; echo "nb1024 rc=$?"
tail -3 gpurun_out/r02_t_nb1024.log
