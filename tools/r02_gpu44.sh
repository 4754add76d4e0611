#!/bin/bash
# TC4 (multicast clusters of two pairs) vs TC2 on the first paired bulk launch (ncu)
cd "$(dirname "$0")/.."
o=gpurun_out/r02ap
mkdir -p $o
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-check"
MPCR_TC4=1 timeout 600 $CMD > $o/plain.log 2>&1; echo "plain rc=$?"
MPCR_TC4=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 4 -c 1 -o $o/tc4_bulk $CMD > $o/ncu_tc4.log 2>&1; echo "ncu tc4 rc=$?"
