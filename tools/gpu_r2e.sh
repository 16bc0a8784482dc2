mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sweep_variants.py -m gpu -q -p no:cacheprovider > gpurun_out/gt_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_e.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
RCG_GRID_SPMV=0 timeout 900 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench_nogrid.json 2> gpurun_out/bench_nogrid.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
