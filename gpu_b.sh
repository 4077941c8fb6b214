make -C paper_2105_10332_b200/csrc -j8 > /dev/null
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "torchrun or multi_device" -p no:cacheprovider > gpurun_out/gt_dist.log 2>&1; echo "dist rc=$?"
tail -30 gpurun_out/gt_dist.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/gt_full.log 2>&1; echo "full rc=$?"
tail -15 gpurun_out/gt_full.log
