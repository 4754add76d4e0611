#!/bin/bash
# ncu --set full of the step-0 FP16 bulk update at n=131072 (pair-kernel launch 2
# of the eager factorization: 7750 tiles), after a plain run of the same command.
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 600 $CMD > $OUT/prof_plain_g8.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 2 -c 1 \
    -o $OUT/tc2_131k_g8 $CMD > $OUT/ncu_full_131k_g8.log 2>&1
echo fin
