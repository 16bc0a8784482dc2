# dev: the default bench line N times (variance)
mkdir -p gpurun_out
for i in $(seq 1 ${N:-3}); do timeout 900 python bench.py ${ARGS:---no-variants --no-cpu-baseline} > gpurun_out/br_$i.json 2> gpurun_out/br_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/br_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['achieved'])" >> gpurun_out/br.log 2>&1; done
