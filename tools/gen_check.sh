# dev: device generator parity + sweep variants + multicolour variant timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_generators.py tests/test_gpu_sweep_cluster.py -x -q -s > gpurun_out/gen_test.log 2>&1; echo "rc=$?" >> gpurun_out/gen_test.log
RCG_SWEEP_CLUSTER=2 timeout 600 python tools/config_probe.py c2 --mc --batch 0 > gpurun_out/gen_probe.log 2>&1
