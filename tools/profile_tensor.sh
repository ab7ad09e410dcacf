#!/bin/bash
# Run under gpurun.  (1) per-launch device times of one bench step (ncu
# gpu__time_duration, cold-cache and serialised: compare shares), (2) one
# `ncu --set full` capture of the main tensor scan launch.
set -e
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-q-sweep > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:tensor_scan_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG -f \
    timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-q-sweep > gpurun_out/prof_$TAG.log 2>&1
