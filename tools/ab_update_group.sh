#!/bin/bash
# A/B of the FP16 update-tile order (MPCR_UPDATE_GROUP: 1 = tile-column order).
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_tile.py -q -x -p no:cacheprovider > $OUT/ab_ug_t.log 2>&1; echo EXIT $? >> $OUT/ab_ug_t.log
for g in 1 8 16 1 8 16; do
  MPCR_UPDATE_GROUP=$g timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_ug64_$g.log 2>&1
done
for g in 1 8 16 8; do
  MPCR_UPDATE_GROUP=$g timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_ug131_$g.log 2>&1
done
echo fin
