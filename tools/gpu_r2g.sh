mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gt_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_g.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
for cm in 2 3 4 6; do
  echo "cmul $cm" >> gpurun_out/cmul.log
  RCG_BSWEEP_CMUL=$cm timeout 300 python tools/profile_batched.py c3 24 6 deflation >> gpurun_out/cmul.log 2>&1
done
