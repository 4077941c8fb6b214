#!/bin/bash
# Launch list (per-launch device time, ncu serialises launches and runs them
# cold-cache: compare SHARES, not absolutes) of a short bench run at the
# bench's per-GPU size (8192^2, b16; 140 requested steps = 20 swept cycles):
#   bash profiles/launch_list.sh <tag>     (under gpurun, from the repo root)
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra > gpurun_out/launches_bench_$TAG.log 2>&1
tail -2 gpurun_out/launches_bench_$TAG.log
