# dev: sweep latency vs resident CTAs per SM (RCG_SWEEP_BPS) and poll backoff
for cfg in c1 c2; do
for bps in 1 4 16; do for bo in 0 20; do
RCG_SWEEP_BPS=$bps RCG_SWEEP_BACKOFF_NS=$bo timeout 120 python tools/sweep_tune.py $cfg 20 2>&1 | tail -1
done; done; done
