# dev: batched alpha/beta history + per-solve Lanczos condest in the sequence
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sequence.py tests/test_gpu_batch.py -x -q > gpurun_out/kap_test.log 2>&1; echo "rc=$?" >> gpurun_out/kap_test.log
