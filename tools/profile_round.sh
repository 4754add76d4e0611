#!/bin/bash
# Runs on the GPU box: plain bench, then the ncu launch list of the same
# command, then one full capture of the dominant kernel.  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > $OUT/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
$CMD > $OUT/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 40 -c 1 -o $OUT/tc_full $CMD > $OUT/ncu_full.log 2>&1
echo done
