#!/bin/bash
# A/B of L2 evict_first hints on the pair kernel's C traffic (MPCR_C_EVICT_FIRST),
# then an ncu capture of the n=131072 step-0 bulk launch with the hints on.
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_tile.py tests/test_gpu_linalg.py -q -x -p no:cacheprovider > $OUT/ab_ce_t.log 2>&1; echo EXIT $? >> $OUT/ab_ce_t.log
for e in 0 1 0 1; do
  MPCR_C_EVICT_FIRST=$e timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_ce64_$e.log 2>&1
done
for e in 0 1 0 1; do
  MPCR_C_EVICT_FIRST=$e timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/ab_ce131_$e.log 2>&1
done
for e in 0 1; do
  MPCR_C_EVICT_FIRST=$e timeout 120 python bench.py --workload gemm --prec half --n 16384 --beta 1 --steps 5 --warmup 3 >> $OUT/ab_ce_gemm_$e.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 2 -c 1 \
    -o $OUT/tc2_131k_ce $CMD > $OUT/ncu_full_131k_ce.log 2>&1
echo fin
