mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweep_variants.py tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider > gpurun_out/gt_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_d.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --impl reference --config c1 --steps 3 --warmup 3 > gpurun_out/bench_ref_c1.json 2> gpurun_out/bench_ref_c1.err
bash tools/prof_c3.sh
