# dev: the sequence step on the other BASELINE configs (C1, C3, C5) and the reference arm on each
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c3 c5}; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-variants > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?" >> gpurun_out/all_configs.log
  timeout 900 python bench.py --impl reference --config $c --steps 1 --warmup 1 > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err
  echo "$c ref rc=$?" >> gpurun_out/all_configs.log
done
