# dev: locate the crash of the c5 loopback sequence (faulthandler stack)
mkdir -p gpurun_out
timeout 300 python -X faulthandler -m pytest tests/test_gpu_dist.py -x -q -k "sequence and c5" -p no:cacheprovider > gpurun_out/segv.log 2>&1; echo "rc=$?" >> gpurun_out/segv.log
