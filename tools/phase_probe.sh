# dev: batch vs concurrent streams
for conc in batch 9 1; do
RCG_CONCURRENCY=$conc timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$conc','value',d['value'],'ms',d['ms_per_step'],d['phases_ms_untimed_step'], {k.split()[0]+k.split()[1]:v['avg_us'] for k,v in d['kernels'].items()})"
done
