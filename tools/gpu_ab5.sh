mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab5.log; env "$@" timeout 600 python tools/profile_batched.py c3 24 20 none >> gpurun_out/ab5.log 2>&1; }
run A=default
run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_exp1.so
run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_exp2.so
run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_exp3.so
run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_exp3.so RCG_BSWEEP_VW=4
run RCG_BSWEEP_CMUL=4
run RCG_BSWEEP_CMUL=2
