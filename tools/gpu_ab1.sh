# dev: A/B of the sweep dependency chunk (ordered consume; all parents in flight in the backward sweep)
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab1.log; env "$@" RS=1,24 timeout 600 python tools/batch_probe.py c3 >> gpurun_out/ab1.log 2>&1; }
run A=default
run RCG_BSWEEP_CH=4 RCG_SWEEP_CH=8
run RCG_BSWEEP_CH=7
run RCG_BSWEEP_CH=13 RCG_BSWEEP_VW=4
run RCG_SWEEP_BPS=2
run RCG_SWEEP_BPS=3
run RCG_BSWEEP_CMUL=1
run RCG_BSWEEP_CMUL=2
run RCG_BSWEEP_CH=7 RCG_BSWEEP_VW=4
run RCG_SWEEP_CH=16
