mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_sequence.py -m gpu -q -p no:cacheprovider > gpurun_out/gt_h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_h.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
RCG_WTY=0 timeout 900 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench_nowty.json 2> gpurun_out/bench_nowty.err
