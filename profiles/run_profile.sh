#!/bin/bash
# Reproduces the profiles/ captures on one B200 (run under gpurun from the repo root).
#   bash profiles/run_profile.sh <tag>
# 1) launch list (per-launch device time, cold-cache, serialised) of a short bench run
# 2) one `ncu --set full` capture of an Octahedron phase launch (steady state) at the
#    bench's per-GPU size, 8192^2 b16, and of the standard heat step
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra > $OUT/launches_bench_$TAG.log 2>&1
# steady-state Octahedron launches are the 4th, 7th, ... swept_phase launches of a solve
ncu --set full --clock-control none --import-source on -k regex:swept_phase_kernel -s 9 -c 1 \
    -o $OUT/prof_oct_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
    > $OUT/prof_oct_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:std_step_kernel -s 5 -c 1 \
    -o $OUT/prof_std_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu \
    > $OUT/prof_std_$TAG.log 2>&1
ls -la $OUT
