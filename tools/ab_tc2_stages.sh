set -x
MPCR_TC2_STAGES=6 timeout 400 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_tile.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/ab_t6.log 2>&1; echo EXIT $? >> gpurun_out/ab_t6.log
for st in 5 6 5 6; do
  for n in 8192 16384; do
    MPCR_TC2_STAGES=$st timeout 120 python bench.py --workload gemm --prec half --n $n --steps 5 --warmup 3 >> gpurun_out/ab_gemm_$st.log 2>&1
  done
  MPCR_TC2_STAGES=$st timeout 120 python bench.py --workload gemm --prec half --n 16384 --beta 1 --steps 5 --warmup 3 >> gpurun_out/ab_gemm_$st.log 2>&1
  MPCR_TC2_STAGES=$st timeout 300 python bench.py --n 65536 --steps 3 --warmup 3 --no-cpu --no-e2e >> gpurun_out/ab_c64_$st.log 2>&1
done
for st in 5 6; do
  MPCR_TC2_STAGES=$st timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> gpurun_out/ab_c131_$st.log 2>&1
done
echo fin
