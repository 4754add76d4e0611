#!/bin/bash
cd "$(dirname "$0")/.."
o=gpurun_out/r02as
mkdir -p $o
ncu --set full --clock-control none --import-source on -k regex:matern -c 1 -o $o/prof_matern python tools/oz_insitu.py 65536 > $o/ncu.log 2>&1; echo "ncu rc=$?"
