# dev: multi-GPU slab tests (loopback + NCCL world 1), bounded
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist_test.log 2>&1; echo "rc=$?" >> gpurun_out/dist_test.log
