#!/bin/bash
# ncu launch list (per-launch gpu__time_duration, serialised, cold cache) of the default
# n=131072 bench command, after a plain run of the same command.  Outputs in gpurun_out/.
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 600 $CMD > $OUT/ll_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_131k.csv $CMD > $OUT/ll_ncu.log 2>&1
echo "ncu rc=$?"
gzip -kf $OUT/launches_131k.csv
echo fin
