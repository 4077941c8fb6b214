#!/bin/bash
# Reproduces the profiles/ evidence on one B200 (run under gpurun from the repo root):
#   bash profiles/run_profile.sh <tag>
# 1) launch list (per-launch device time; ncu serialises launches and runs them
#    cold-cache, so compare SHARES, not absolutes) of a short bench run at the
#    bench's per-GPU size (8192^2, b16; 140 requested steps = 20 swept cycles)
# 2) ncu --set full of one steady-state Octahedron launch and one standard step
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu > $OUT/launches_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:swept_heat -s 9 -c 1 \
    -o $OUT/prof_oct_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
    > $OUT/prof_oct_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:std_heat -s 5 -c 1 \
    -o $OUT/prof_std_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu \
    > $OUT/prof_std_$TAG.log 2>&1
ls -la $OUT
