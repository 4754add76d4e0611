#!/bin/bash
# A/B of the pair kernel's unit assignment (MPCR_UNIT_STRIDED=1: grid-stride),
# then an ncu capture of the n=131072 step-0 bulk launch with the default.
OUT=gpurun_out
timeout 400 python -m pytest tests/test_gpu_tile.py tests/test_gpu_linalg.py -q -x -p no:cacheprovider > $OUT/ab_uo_t.log 2>&1; echo EXIT $? >> $OUT/ab_uo_t.log
grep -q "EXIT 0" $OUT/ab_uo_t.log || exit 1
for e in 1 0 1 0; do
  MPCR_UNIT_STRIDED=$e timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_uo64_$e.log 2>&1
done
for e in 1 0 1 0; do
  MPCR_UNIT_STRIDED=$e timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_uo131_$e.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 2 -c 1 \
    -o $OUT/tc2_131k_uo $CMD > $OUT/ncu_full_131k_uo.log 2>&1
echo fin
