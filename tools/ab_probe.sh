# dev: A/B of an alternative build (tools/ab/$LIB) against the in-tree library on the C2 probe + bench
for lib in "" "$LIB"; do
  if [ -n "$lib" ]; then export RCG_LIB_PATH=tools/ab/$lib; else unset RCG_LIB_PATH; fi
  echo "lib=${lib:-tree}"
  RS=${RS:-1,4,12} timeout 300 python tools/batch_probe.py c2
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'],d['phases_ms_untimed_step'])"
done
