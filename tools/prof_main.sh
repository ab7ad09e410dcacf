#!/bin/bash
# Run under gpurun: one `ncu --set full` capture of one tensor scan launch, tag $1;
# $2 = launches to skip (1: the main scan after the probe, 0: the probe).
TAG=${1:-dev}
SKIP=${2:-1}
ncu --set full --clock-control none --import-source on \
    -k regex:tensor_scan_kernel -s $SKIP -c 1 -o gpurun_out/prof_$TAG -f \
    timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-q-sweep > gpurun_out/prof_$TAG.log 2>&1
echo "ncu rc=$?"
