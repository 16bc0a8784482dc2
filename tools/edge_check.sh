# dev: edge cases (bounded)
mkdir -p gpurun_out
timeout 600 python -X faulthandler -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider > gpurun_out/edge_test.log 2>&1; echo "rc=$?" >> gpurun_out/edge_test.log
