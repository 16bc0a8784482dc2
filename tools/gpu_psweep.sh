# dev: pencil sweep correctness + timing (logs under gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_gpu_sweep_variants.py tests/test_gpu_generators.py -m gpu -q -p no:cacheprovider > gpurun_out/ps_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ps_tests.log
for c in c2 c3 c4; do
  for m in 0 5; do
    RCG_SWEEP_CLUSTER=$m timeout 300 python tools/sweep_tune.py $c 10 >> gpurun_out/ps_tune.log 2>&1
  done
done
echo done >> gpurun_out/ps_tune.log
