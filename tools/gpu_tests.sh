# dev: selected GPU test files (bounded), e.g. bash tools/gpu_tests.sh tests/test_bridge.py tests/test_gpu_sequence.py
mkdir -p gpurun_out
timeout 2400 python -X faulthandler -m pytest "$@" -m gpu -q -p no:cacheprovider -x > gpurun_out/gt_sel.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gt_sel.log
