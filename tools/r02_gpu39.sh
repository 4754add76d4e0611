#!/bin/bash
# INT8-digit kernel at the final code: dense 8192^3 FP16 x FP16 -> FP64 and an in-situ bulk launch
cd "$(dirname "$0")/.."
o=gpurun_out/r02ak
mkdir -p $o
CMD="python bench.py --workload gemm --prec half --cprec double --n 8192 --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > $o/plain.json 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none -k regex:"oz_gemm" -s 1 -c 1 -o $o/prof_oz_dense $CMD > $o/ncu_dense.log 2>&1; echo "ncu dense rc=$?"
ncu --set full --clock-control none -k regex:"oz_gemm" -s 40 -c 8 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_insitu.log 2>&1; echo "ncu insitu rc=$?"
