set -u
TAG=$1
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:swept_heat -s 9 -c 1 \
    -o gpurun_out/prof_oct_$TAG python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/prof_oct_$TAG.log 2>&1
tail -2 gpurun_out/prof_oct_$TAG.log
