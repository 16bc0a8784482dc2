# dev: A/B of the sweep consume order / chunk against the previous library
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab2.log; env "$@" timeout 600 python tools/batch_probe.py c3 >> gpurun_out/ab2.log 2>&1; }
run RS=1,24 RCG_LIB_PATH=$PWD/paper_2203_08498_b200/librcg_old.so
run RS=1 RCG_SWEEP_ORD=0 RCG_SWEEP_CH=8
run RS=1 RCG_SWEEP_ORD=0 RCG_SWEEP_CH=16
run RS=1 RCG_SWEEP_ORD=0 RCG_SWEEP_CH=16 RCG_SWEEP_BPS_BWD=2
run RS=1 RCG_SWEEP_ORD=1 RCG_SWEEP_CH=16 RCG_SWEEP_BPS_BWD=2
run RS=1 RCG_SWEEP_ORD=1 RCG_SWEEP_CH=8 RCG_SWEEP_BPS_BWD=2
run RS=1 RCG_SWEEP_ORD=0 RCG_SWEEP_CH=8 RCG_SWEEP_BPS_BWD=2
run RS=12,24 RCG_BSWEEP_CH=4
run RS=12,24 RCG_BSWEEP_CH=4 RCG_BSWEEP_VW=4
run RS=12,24 RCG_BSWEEP_CH=4 RCG_BSWEEP_VW=2
run RS=24 RCG_BSWEEP_CH=4 RCG_BSWEEP_CMUL=4
run RS=24 RCG_BSWEEP_CH=4 RCG_BSWEEP_CMUL=2
