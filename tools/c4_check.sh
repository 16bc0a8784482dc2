# dev: lean distributed recycling parity, then C4 through the row-slab path on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/c4s_test.log 2>&1; echo "rc=$?" >> gpurun_out/c4s_test.log
timeout 2400 python tools/c4_slabs.py 1 > gpurun_out/c4_slabs.json 2> gpurun_out/c4_slabs.err; echo "c4 slabs rc=$?" >> gpurun_out/c4_slabs.err
