mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_dist_host.py tests/test_bench_contract.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py tests/test_gpu_batch.py tests/test_bridge.py -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gt_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_c.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
RCG_BSWEEP_VW=4 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_vw4.json 2> gpurun_out/bench_vw4.err
