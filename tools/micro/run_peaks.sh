#!/bin/bash
# Pipe peaks for the blended roofline (run on a B200 via gpurun), with the
# clocks sampled while they run.  Binaries are built here:
#   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc_peak tc_peak.cu
#   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
out=$(realpath -m "${1:-gpurun_out/r02_peaks}")
cd "$(dirname "$0")"
mkdir -p "$(dirname "$out")"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 200 > "$out.clocks.csv" &
smi=$!
./tc_peak 4 > "$out.txt" 2>&1
./fp64_peak >> "$out.txt" 2>&1
kill $smi
cat "$out.txt"
