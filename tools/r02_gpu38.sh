#!/bin/bash
# final check at HEAD: full GPU suite, smoke, default bench
cd "$(dirname "$0")/.."
o=gpurun_out/r02aj
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $o/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $o/smoke.txt
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench_default.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['value'], d['blended_roofline']['frac'], d['roofline']['frac'], d['accuracy']['sampled_backward_error'])"
