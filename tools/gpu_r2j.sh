# dev: round-2 re-entry checkpoint -- default bench (C3), reference arm, ncu launch list of the
# bench command, ncu --set full of the C3 hot kernels (CSV summaries come back), smoke
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu.log
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_b_sweepc|k_b_spmv|k_b_tallt|k_b_wty|k_b_deflate|k_b_pupdate|k_b_xr|k_b_rho|k_sweep|k_spmv_pq|k_pupdate|k_xr" -c 40 \
  -o /tmp/ncu/prof_c3 -f python tools/profile_batched.py c3 24 2 deflation > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3.log
ncu -i /tmp/ncu/prof_c3.ncu-rep --page raw --csv > gpurun_out/prof_c3_raw.csv 2>/dev/null
ls -la gpurun_out /tmp/ncu >> gpurun_out/ncu_c3.log
