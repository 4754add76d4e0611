#!/bin/bash
# Runs on the GPU box: GPU tests + smoke, the default bench line (n=131072),
# then one ncu --set full capture of the largest FP16 bulk-update launch of the
# first (eager) factorization of the same command.  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/tgpu.log 2>&1; echo EXIT $? >> $OUT/tgpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo EXIT $? >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --n 65536 > $OUT/bench_65536.json 2> $OUT/bench_65536.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
MPCR_DEBUG_TC=1 timeout 600 $CMD > $OUT/prof_plain.log 2> $OUT/prof_plain.err || { echo "plain run failed"; exit 1; }
IDX=$(python - <<'PY'
import re
best=None
for i,l in enumerate(open("gpurun_out/prof_plain.err")):
    m=re.match(r"\[mpcr\] tc2 launch (\d+): C half, (\d+) problem", l)
    if not m: continue
    idx,cnt=int(m.group(1)),int(m.group(2))
    if idx>=380: break
    if best is None or cnt>best[1]: best=(idx,cnt)
print(best[0], best[1])
PY
)
echo "capture: $IDX" > $OUT/ncu131_idx.txt
set -- $IDX
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s $1 -c 1 \
    -o $OUT/tc2_131k $CMD > $OUT/ncu_full_131k.log 2>&1
echo fin
