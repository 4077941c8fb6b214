#!/bin/bash
# ncu --set full of one steady-state swept cycle (Octahedron, YBridge, XBridge
# launches 9..11) of the heat bench workload (8192^2, b16):
#   bash profiles/prof_col.sh <tag>      (under gpurun, from the repo root)
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:swept_heat -s 9 -c 3 \
    -o gpurun_out/prof_cycle_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/prof_cycle_$TAG.log 2>&1
tail -3 gpurun_out/prof_cycle_$TAG.log
