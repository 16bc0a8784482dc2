mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist_host.py tests/test_gpu_batch.py tests/test_gpu_golden.py tests/test_bridge.py -m gpu -q -p no:cacheprovider > gpurun_out/gt_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_b.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
