# dev: GPU suite + C2 kernel probe + short bench (logs under gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt.log
RS=${RS:-1,4,12} timeout 300 python tools/batch_probe.py c2 > gpurun_out/probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
