#!/bin/bash
# A/B of the tile-column write-back stream (MPCR_WB_ASYNC: 0 = on the bulk stream).
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tile.py -q -x -p no:cacheprovider > $OUT/ab_wb_t.log 2>&1; echo EXIT $? >> $OUT/ab_wb_t.log
for w in 1 0 1 0; do
  MPCR_WB_ASYNC=$w timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_wb131_$w.log 2>&1
done
for w in 1 0 1 0; do
  MPCR_WB_ASYNC=$w timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_wb64_$w.log 2>&1
done
echo fin
