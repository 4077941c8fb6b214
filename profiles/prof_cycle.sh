#!/bin/bash
# ncu --set full of one steady-state swept cycle (Octahedron, YBridge, XBridge
# = heat launches 9..11) of the bench grid (8192^2) at block B:
#   bash profiles/prof_cycle.sh <tag> <B>      (under gpurun, from the repo root)
set -u
TAG=${1:-r02}
B=${2:-16}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:swept_heat -s 9 -c 3 \
    -o gpurun_out/prof_cycle_b${B}_$TAG python bench.py --block $B --req-steps 140 --steps 1 --warmup 3 --no-cpu \
    --no-extra > gpurun_out/prof_cycle_b${B}_$TAG.log 2>&1
tail -3 gpurun_out/prof_cycle_b${B}_$TAG.log
