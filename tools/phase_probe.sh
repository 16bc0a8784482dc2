# dev: concurrency vs shared-memory carveout
for co in -1 50 100; do
RCG_CARVEOUT=$co RCG_CONCURRENCY=9 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('carveout',$co,'value',d['value'],'ms',d['ms_per_step'],{k:v for k,v in d['phases_ms_untimed_step'].items() if k!='accelerated_iterations'}, {k.split()[0]+k.split()[1]:v['avg_us'] for k,v in d['kernels'].items()})"
done
