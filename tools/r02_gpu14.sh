#!/bin/bash
# oz slicer: digits of the needed planes only; tests, bench, in-situ captures, launch list
cd "$(dirname "$0")/.."
o=gpurun_out/r02l
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_linalg.py -q -x -k "half_to_double or int8 or digit" > $o/t_linalg.log 2>&1; echo "linalg-oz rc=$?"; tail -2 $o/t_linalg.log
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_dist_sim.py -q -x > $o/t_tile.log 2>&1; echo "tile rc=$?"; tail -2 $o/t_tile.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['clocks']['sm_mhz'], d['accuracy']['sampled_backward_error'], d['accuracy']['leading_block_bitwise_equal'], {k:round(v['ms'],1) for k,v in d['breakdown']['classes'].items()})"
timeout 600 python tools/trace_chol.py 131072 1024 $o/trace.csv > $o/trace.txt 2>&1; echo "trace rc=$?"; cat $o/trace.txt
ncu --set full --clock-control none --import-source on -k regex:"oz_slice" -s 20 -c 1 -o $o/prof_slice_insitu python tools/oz_insitu.py 65536 > $o/ncu_slice.log 2>&1; echo "ncu slice rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_65536.csv python tools/oz_insitu.py 65536 > $o/ncu_ll.log 2>&1; echo "ncu ll rc=$?"
python tools/launch_summary.py $o/launches_65536.csv | head -40
