# dev: bench value vs concurrent solves and sweep residency
for conc in 3 9; do for bps in 0 1; do
RCG_CONCURRENCY=$conc RCG_SWEEP_BPS=$bps timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conc',$conc,'bps',$bps,'value',d['value'],'ms',d['ms_per_step'],d['phases_ms_untimed_step'])"
done; done
