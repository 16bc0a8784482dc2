mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gt_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_f.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
