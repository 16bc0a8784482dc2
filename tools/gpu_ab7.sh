mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab7.log; env "$@" >> gpurun_out/ab7.log 2>&1; }
run A=default timeout 600 python tools/profile_batched.py c3 24 20 deflation
run RS=1,16 timeout 600 python tools/batch_probe.py c3
run RS=1,4,9,12 timeout 600 python tools/batch_probe.py c2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > gpurun_out/ab7_tests.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_ab7.json 2> gpurun_out/bench_ab7.err
