# dev: batched kernels after the deflate / pupdate unroll and residency changes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sequence.py -x -q > gpurun_out/bprof_test.log 2>&1; echo "rc=$?" >> gpurun_out/bprof_test.log
for c in c3 c5 c2; do for k in sc deflation; do
  echo "== $c $k" >> gpurun_out/bprof_live.log
  timeout 600 python tools/profile_batched.py $c 12 3 $k >> gpurun_out/bprof_live.log 2>&1
done; done
