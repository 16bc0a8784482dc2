# dev: sweep + spmv timing
for cfg in c1 c2 c2mc c3 c5; do
timeout 300 python tools/sweep_tune.py $cfg 10 2>&1 | tail -1
done
