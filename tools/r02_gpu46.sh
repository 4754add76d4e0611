#!/bin/bash
# Matern FP16 generator: fast path for tiny values, shift indexing, walking upper pointer
cd "$(dirname "$0")/.."
o=gpurun_out/r02ar
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_nll.py tests/test_gpu_casts_ew.py -q -x -k "matern or fill or nll" > $o/t.log 2>&1; echo "tests rc=$?"; tail -2 $o/t.log
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:matern -c 1 python tools/oz_insitu.py 65536 > $o/ncu_matern.log 2>&1; echo "ncu rc=$?"; grep -E "duration|bytes_write|inst_executed" $o/ncu_matern.log | head -4
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-check > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1), round(d['ms_per_step'],1))"
done
