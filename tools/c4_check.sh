# dev: lean-sequence parity, then C4 on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sequence.py -x -q > gpurun_out/c4_test.log 2>&1; echo "rc=$?" >> gpurun_out/c4_test.log
timeout 1800 python tools/c4_run.py 40 > gpurun_out/c4_run.json 2> gpurun_out/c4_run.err; echo "c4 rc=$?" >> gpurun_out/c4_run.err
