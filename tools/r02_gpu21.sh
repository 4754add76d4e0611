#!/bin/bash
# trace + oz capture after the FP32-digit change
cd "$(dirname "$0")/.."
o=gpurun_out/r02s
mkdir -p $o
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 60 -c 6 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
