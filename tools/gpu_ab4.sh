mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab4.log; env "$@" timeout 600 python tools/profile_batched.py c3 24 20 none >> gpurun_out/ab4.log 2>&1; }
run A=default
run RCG_BSWEEP_CA=1
run RCG_BSWEEP_CH=7
run RCG_BSWEEP_CH=7 RCG_BSWEEP_CA=1
run RCG_BSWEEP_CA=1 RCG_BSWEEP_VW=4
run RCG_BSWEEP_CA=1 RCG_BSWEEP_VW=2
echo "== single" >> gpurun_out/ab4.log
RS=1,12 timeout 600 python tools/batch_probe.py c3 >> gpurun_out/ab4.log 2>&1
RS=12 RCG_BSWEEP_CA=1 timeout 600 python tools/batch_probe.py c3 >> gpurun_out/ab4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q -p no:cacheprovider > gpurun_out/ab4_tests.log 2>&1
RCG_BSWEEP_CA=1 timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/ab4_tests.log 2>&1
