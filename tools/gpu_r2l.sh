# dev: A/B of the batched chunk-lane sweeps' entry-record prefetch (RCG_BSWEEP_PF: 0 off, 1 L2, 2 L1,
# +4 backward only) on C3 at RT 24, then the bench with the candidates
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/ab_pf.log; env "$@" >> gpurun_out/ab_pf.log 2>&1; }
for pf in 0 2 1 6 10 8; do
  run RCG_BSWEEP_PF=$pf timeout 600 python tools/profile_batched.py c3 24 20 deflation
done
run RCG_BSWEEP_PF=2 RCG_BSWEEP_VW=4 timeout 600 python tools/profile_batched.py c3 24 20 deflation
run RCG_BSWEEP_PF=2 RCG_BSWEEP_CMUL=4 timeout 600 python tools/profile_batched.py c3 24 20 deflation
run RCG_BSWEEP_PF=2 timeout 600 python tools/profile_batched.py c2 12 20 sc
run RCG_BSWEEP_PF=0 timeout 600 python tools/profile_batched.py c2 12 20 sc
RCG_BSWEEP_PF=10 timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pf_tests.log 2>&1
RCG_BSWEEP_PF=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pf2.json 2> gpurun_out/bench_pf2.err
RCG_BSWEEP_PF=10 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pf10.json 2> gpurun_out/bench_pf10.err
RCG_BSWEEP_PF=10 timeout 900 python -m pytest tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pf_tests2.log 2>&1
