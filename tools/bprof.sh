# dev: batched W^T r after the JC / reduction change
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sequence.py -x -q > gpurun_out/bprof_test.log 2>&1; echo "rc=$?" >> gpurun_out/bprof_test.log
for c in c2 c3 c5; do for R in 12 8 4; do
  echo "== $c sc R$R" >> gpurun_out/bprof_live.log
  timeout 600 python tools/profile_batched.py $c $R 3 sc >> gpurun_out/bprof_live.log 2>&1
done; done
