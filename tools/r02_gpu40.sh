#!/bin/bash
# Matern FP16 generator: four-block strips
cd "$(dirname "$0")/.."
o=gpurun_out/r02al
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_nll.py -q -x -k "matern or fill or nll" > $o/t.log 2>&1; echo "tests rc=$?"; tail -2 $o/t.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-check"
timeout 600 $CMD > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],1), d['e2e']['ms_per_step'], d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:matern -c 1 python tools/oz_insitu.py 65536 > $o/ncu_matern.log 2>&1; echo "ncu rc=$?"; grep -E "matern|duration|bytes_write" $o/ncu_matern.log | head -6
