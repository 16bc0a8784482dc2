# dev: the whole GPU suite (bounded)
mkdir -p gpurun_out
timeout 1500 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt.log
