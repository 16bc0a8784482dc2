# dev: sweep timing, level skipping on/off
for cfg in c1 c2 c2mc c3 c5; do
for sk in 0 1; do
RCG_SWEEP_SKIP=$sk timeout 300 python tools/sweep_tune.py $cfg 10 2>&1 | tail -1 | sed "s/^/skip=$sk /"
done; done
