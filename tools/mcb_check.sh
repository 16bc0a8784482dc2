# dev: batched per-level sweeps (parity + multicolour timing)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep_cluster.py tests/test_gpu_batch.py -x -q > gpurun_out/mcb_test.log 2>&1; echo "rc=$?" >> gpurun_out/mcb_test.log
timeout 900 python tools/config_probe.py c2 c3 --mc --batch 8 > gpurun_out/mcb_probe.log 2>&1
