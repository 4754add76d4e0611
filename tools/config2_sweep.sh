#!/bin/bash
# BASELINE.json configs[1]: per-precision GEMM and the six cast directions at
# n = 4096 .. 32768 on one B200 (bench.py lines, one per case).
mkdir -p gpurun_out
for n in 4096 8192 16384 32768; do
  for p in half single double; do
    [ "$p" = "double" ] && [ $n -gt 16384 ] && continue   # FP64 32768^3 takes ~2.7 s per step
    python bench.py --workload gemm --prec $p --n $n --steps 3 --warmup 3 --no-cpu 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'gemm {\"$p\":7s} n={$n:6d} {d[\"value\"]:9.1f} {d[\"unit\"]}  roofline {(d.get(\"roofline\") or {}).get(\"frac\")}')"
  done
done
for n in 8192 32768; do
  for c in double:half double:single single:half half:single half:double single:double; do
    python bench.py --workload cast --cast $c --n $n --steps 5 --warmup 3 --no-cpu 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'cast {\"$c\":14s} n={$n:6d} {d[\"value\"]:9.1f} {d[\"unit\"]}  roofline {(d.get(\"roofline\") or {}).get(\"frac\")}')"
  done
done
