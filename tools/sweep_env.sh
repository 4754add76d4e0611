#!/bin/bash
# usage: tools/sweep_env.sh "VAR=a VAR2=b" "VAR=c" ...   (each arg one config)
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/sweep.json"))
print(f"{sys.argv[1]:40s} {d['value']:7.1f} TF/s {d['ms_per_step']:7.1f} ms  blended {d['blended_roofline']['frac']:.3f}")
PY
done
