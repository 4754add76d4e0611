#!/bin/bash
# tests after the TRSM K-range change, bench, chain, config lines, ncu evidence
cd "$(dirname "$0")/.."
o=gpurun_out/r02e
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_dist_sim.py tests/test_gpu_tile.py -q -x > $o/t_tile.log 2>&1; echo "tile+dist rc=$?"; tail -2 $o/t_tile.log
timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain.txt 2>&1; echo "chain rc=$?"; tail -1 $o/chain.txt
B="python bench.py"
for d in half:single single:half half:double double:half single:double double:single; do
  for n in 8192 32768; do
    timeout 300 $B --workload cast --cast $d --n $n --steps 20 --warmup 5 $( [ $n = 32768 ] && echo --no-cpu ) > $o/cast_${d/:/_}_$n.json 2>> $o/err.log; echo "cast $d $n rc=$?"
  done
done
timeout 300 $B --workload gemm --prec half --n 8192 --steps 20 --warmup 5 --no-cpu > $o/gemm_half_8192.json 2>> $o/err.log; echo "gemm rc=$?"
timeout 300 $B --workload gemm --prec single --n 2048 --steps 50 --warmup 5 > $o/gemm_single_2048.json 2>> $o/err.log; echo "gemm1 rc=$?"
timeout 300 $B --workload gemm --prec single --n 8192 --steps 20 --warmup 5 --no-cpu > $o/gemm_single_8192.json 2>> $o/err.log; echo "gemm32 rc=$?"
# ncu evidence (each after its plain run above exited 0)
timeout 300 python tools/prof_kernels.py all > $o/prof_plain.txt 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:convert --csv \
    --log-file $o/ncu_casts.csv python tools/prof_kernels.py casts > $o/ncu_casts.log 2>&1; echo "ncu casts rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dmma_gemm -s 2 -c 1 -o $o/prof_dmma python tools/prof_kernels.py dmma > $o/ncu_dmma.log 2>&1; echo "ncu dmma rc=$?"
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 2 -c 1 -o $o/prof_oz python tools/prof_kernels.py ozaki > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
ncu --set full --clock-control none --import-source on -k regex:matern_tiles -s 2 -c 1 -o $o/prof_matern python tools/prof_kernels.py matern > $o/ncu_matern.log 2>&1; echo "ncu matern rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o $o/prof_f16 python tools/prof_kernels.py f16 > $o/ncu_f16.log 2>&1; echo "ncu f16 rc=$?"
