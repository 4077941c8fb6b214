set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -C paper_2105_10332_b200/csrc -j8 > /dev/null
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r02a.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_r02a.log
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r02a.json
timeout 600 bash profiles/prof_cycle.sh r02a 32
timeout 600 bash profiles/prof_euler.sh r02a
ls -la gpurun_out
