#!/bin/bash
# Round-2 evidence at the final code: GPU test suite, default bench line (e2e + CPU
# baseline), reference arm, ncu launch list of the bench command, one ncu --set full
# capture of the first paired bulk tcgen05 launch, critical-chain timing.
cd "$(dirname "$0")/.."
o=gpurun_out/r02final
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.txt
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?"; tail -c 600 $o/bench_default.json
timeout 900 python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_reference.err; echo "ref rc=$?"; tail -c 300 $o/bench_reference.json
timeout 600 python tools/chain_time.py 131072 1024 > $o/chain.txt 2>&1; echo "chain rc=$?"; tail -4 $o/chain.txt
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-check"
timeout 600 $CMD > $o/ll_plain.log 2>&1; echo "plain rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_n131072.csv $CMD > $o/ll_ncu.log 2>&1; echo "ncu ll rc=$?"
python tools/launch_summary.py $o/launches_n131072.csv "n=131072 default bench command (steps 1, warmup 1), ncu launch list" > $o/launch_summary.txt 2>&1; head -20 $o/launch_summary.txt
gzip -kf $o/launches_n131072.csv
# first tcgen05 launch longer than 5 ms = the first paired bulk update
SKIP=$(python - <<PY
import csv
rows=list(csv.reader(open("$o/launches_n131072.csv")))
h=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
c=rows[h]; ki,vi,ui=c.index("Kernel Name"),c.index("Metric Value"),c.index("Metric Unit")
n=0
for r in rows[h+1:]:
    if len(r)<=vi or "gemm_tc2_kernel" not in r[ki]: continue
    v=float(r[vi].replace(",",""))*{"ns":1e-6,"us":1e-3,"usecond":1e-3,"nsecond":1e-6,"ms":1.0,"msecond":1.0}.get(r[ui],1e-6)
    if v>5.0: print(n); break
    n+=1
PY
)
echo "bulk launch index $SKIP"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s $SKIP -c 1 -o $o/tc2_bulk_n131072 $CMD > $o/ncu_full.log 2>&1; echo "ncu full rc=$?"
