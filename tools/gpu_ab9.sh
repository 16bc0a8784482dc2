mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab9.log; env "$@" >> gpurun_out/ab9.log 2>&1; }
run A=default timeout 600 python tools/profile_batched.py c3 24 20 deflation
run A=default timeout 600 python tools/profile_batched.py c3 16 20 sc
run A=default timeout 600 python tools/profile_batched.py c2 12 20 sc
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_dist.py tests/test_gpu_dist_host.py tests/test_gpu_sequence.py tests/test_gpu_golden.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider > gpurun_out/ab9_tests.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_ab9.json 2> gpurun_out/bench_ab9.err
