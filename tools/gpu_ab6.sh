mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab6.log; env "$@" >> gpurun_out/ab6.log 2>&1; }
run A=default timeout 600 python tools/profile_batched.py c3 24 20 none
run RCG_BSWEEP_VW=4 timeout 600 python tools/profile_batched.py c3 24 20 none
run RCG_BSWEEP_VW=2 timeout 600 python tools/profile_batched.py c3 24 20 none
run RCG_BSWEEP_CMUL=2 timeout 600 python tools/profile_batched.py c3 24 20 none
run RS=1,8,12,16 timeout 600 python tools/batch_probe.py c3
run RS=1,4,9,12 timeout 600 python tools/batch_probe.py c2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_icfactor.py tests/test_gpu_edges.py tests/test_gpu_sweep_variants.py -m gpu -x -q -p no:cacheprovider > gpurun_out/ab6_tests.log 2>&1
