#!/bin/bash
# Run under gpurun: one `ncu --set full` capture of the main tensor scan launch only
# (the probe launch is -s 1 skipped), tag $1.
TAG=${1:-dev}
ncu --set full --clock-control none --import-source on \
    -k regex:tensor_scan_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG -f \
    timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_$TAG.log 2>&1
echo "ncu rc=$?"
