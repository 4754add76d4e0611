#!/bin/bash
# in-situ oz capture after dynamic scheduling; POTRF phase trace
cd "$(dirname "$0")/.."
o=gpurun_out/r02p
mkdir -p $o
timeout 300 python tools/prof_potrf.py 1024 > $o/potrf_time.txt 2>&1; echo "potrf rc=$?"; tail -3 $o/potrf_time.txt
MPCR_POTRF_TRACE=1 timeout 300 python tools/prof_potrf.py 1024 > $o/potrf_trace.txt 2>&1; echo "potrf trace rc=$?"; grep "potrf trace" $o/potrf_trace.txt | tail -2
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm" -s 40 -c 2 -o $o/prof_oz_insitu python tools/oz_insitu.py 65536 > $o/ncu_oz.log 2>&1; echo "ncu oz rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"potrf_coop" -s 5 -c 1 -o $o/prof_potrf python tools/prof_potrf.py 1024 > $o/ncu_potrf.log 2>&1; echo "ncu potrf rc=$?"
