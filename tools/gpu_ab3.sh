mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab3.log; env "$@" >> gpurun_out/ab3.log 2>&1; }
OLD=RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_old.so
run $OLD timeout 600 python tools/profile_batched.py c3 24 20 deflation
run $OLD timeout 600 python tools/profile_batched.py c3 24 20 none
run $OLD timeout 600 python tools/profile_batched.py c3 19 20 deflation
run RCG_BSWEEP_CH=4 timeout 600 python tools/profile_batched.py c3 24 20 deflation
run RCG_BSWEEP_CH=4 timeout 600 python tools/profile_batched.py c3 24 20 none
run RS=1 RCG_SWEEP_CH=16 RCG_SWEEP_BPS_BWD=2 timeout 600 python tools/batch_probe.py c3
run RS=1 RCG_SWEEP_CH=16 RCG_SWEEP_BPS_BWD=3 timeout 600 python tools/batch_probe.py c3
