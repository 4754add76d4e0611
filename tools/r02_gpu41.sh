#!/bin/bash
# A/B: Matern FP16 generator one-block vs four-block strips, n = 131072 (ncu time + e2e)
cd "$(dirname "$0")/.."
o=gpurun_out/r02am
mkdir -p $o
for v in old new old new; do
  cp tools/ab/lib_matern_$v.so paper_2406_02701_b200/libmpcr_b200.so
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-check > $o/bench.json 2> $o/bench.err
  echo "$v $(python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1), round(d['ms_per_step'],1))")"
done
for v in old new; do
  cp tools/ab/lib_matern_$v.so paper_2406_02701_b200/libmpcr_b200.so
  ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:matern -c 1 python tools/oz_insitu.py 131072 > $o/ncu_$v.log 2>&1
  echo "$v $(grep -E "duration|bytes_write" $o/ncu_$v.log | tr -s ' ' | tr '\n' ' ')"
done
