#!/bin/bash
# config-1/2/5 lines, cast sweep, API tests
cd "$(dirname "$0")/.."
o=gpurun_out/r02c
mkdir -p $o
timeout 600 python -m pytest tests/test_cpp_boundary.py tests/test_gpu_linalg.py -q -x -k "facade or dispatch or large_k" -s > $o/t_api.log 2>&1; echo "api rc=$?"; tail -2 $o/t_api.log
timeout 900 python tools/cast_sweep.py > $o/cast_sweep.jsonl 2> $o/cast_sweep.err; echo "sweep rc=$?"
B="python bench.py"
timeout 300 $B --workload gemm --prec single --n 2048 --steps 10 --warmup 3 > $o/gemm_single_2048.json 2>> $o/err.log; echo "g1 rc=$?"
for pr in half single double; do for n in 8192 16384; do
  timeout 600 $B --workload gemm --prec $pr --n $n --steps 5 --warmup 3 > $o/gemm_${pr}_$n.json 2>> $o/err.log; echo "gemm $pr $n rc=$?"
done; done
timeout 600 $B --workload gemm --prec half --cprec double --n 8192 --steps 5 --warmup 3 > $o/gemm_half_double_8192.json 2>> $o/err.log; echo "gemm h->d rc=$?"
timeout 900 $B --workload gemm --prec half --n 32768 --steps 3 --warmup 3 > $o/gemm_half_32768.json 2>> $o/err.log; echo "gemm h 32768 rc=$?"
timeout 900 $B --workload gemm --prec double --n 32768 --steps 2 --warmup 3 > $o/gemm_double_32768.json 2>> $o/err.log; echo "gemm d 32768 rc=$?"
for d in half:single single:half half:double double:half single:double double:single; do
  timeout 300 $B --workload cast --cast $d --n 8192 --steps 20 --warmup 5 > $o/cast_${d/:/_}_8192.json 2>> $o/err.log; echo "cast $d rc=$?"
done
timeout 1200 $B --workload nll --n 65536 --steps 3 --warmup 3 > $o/nll_65536.json 2>> $o/err.log; echo "nll rc=$?"
