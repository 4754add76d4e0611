#!/bin/bash
# POTRF alone vs CTA count
cd "$(dirname "$0")/.."
o=gpurun_out/r02y
mkdir -p $o
for c in 16 24 32 48 64 96 120; do
  echo "ctas=$c $(MPCR_POTRF_CTAS=$c timeout 300 python tools/prof_potrf.py 1024 2>&1 | grep median)"
  MPCR_POTRF_CTAS=$c MPCR_POTRF_TRACE=1 timeout 300 python tools/prof_potrf.py 1024 2>&1 | grep "potrf trace" | tail -1
done
