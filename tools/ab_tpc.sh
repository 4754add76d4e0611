#!/bin/bash
# Sweep of MPCR_TILES_PER_CTA (bulk GEMM CTAs retire after this many tiles) with the
# wave-contiguous unit assignment, n=131072 and n=65536, interleaved.
OUT=gpurun_out
mkdir -p $OUT
for r in 1 2; do
  for t in 16 24 32 48; do
    MPCR_TILES_PER_CTA=$t timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/tpc131_$t.log 2>&1
  done
done
for t in 16 24 32 48; do
  MPCR_TILES_PER_CTA=$t timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> $OUT/tpc64_$t.log 2>&1
done
echo fin
