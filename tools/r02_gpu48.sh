#!/bin/bash
# Matern FP16 generator: branch-free stores, warp-level fallback queueing
cd "$(dirname "$0")/.."
o=gpurun_out/r02at
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_nll.py tests/test_gpu_casts_ew.py -q -x -k "matern or fill or nll" > $o/t.log 2>&1; echo "tests rc=$?"; tail -2 $o/t.log
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:matern -c 1 python tools/oz_insitu.py 65536 > $o/ncu_matern.log 2>&1; echo "ncu rc=$?"; grep -E "duration|inst_executed" $o/ncu_matern.log | head -4
