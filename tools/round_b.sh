# dev: GPU suite, bench (C2 default), then the other configs
mkdir -p gpurun_out
timeout 1500 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CONFIGS="c3 c5 c1" bash tools/all_configs.sh
