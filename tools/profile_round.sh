#!/bin/bash
# Runs on the GPU box: the default bench line, then (same command, plain run
# first) the ncu launch list, then one full capture each of the two dominant
# kernels (FP16 2-CTA trailing update, INT8-digit FP64 SYRK).  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD \
    > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 150 -c 3 \
    -o $OUT/tc2_full $CMD > $OUT/ncu_full_tc2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm_kernel -s 150 -c 2 \
    -o $OUT/oz_full $CMD > $OUT/ncu_full_oz.log 2>&1
echo done
