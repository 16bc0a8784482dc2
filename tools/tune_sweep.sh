# dev: sweep latency/throughput vs resident CTAs per SM (RCG_SWEEP_BPS)
for cfg in c1 c2 c2mc c3; do
for bps in 2 4 8; do
RCG_SWEEP_BPS=$bps timeout 300 python tools/sweep_tune.py $cfg 10 2>&1 | tail -1
done; done
