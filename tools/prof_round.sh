# dev: this round's profiles -- launch list of the bench command, ncu full capture of the C2 hot kernels
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu.log
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_sweep|k_b_sweepc|spmv_pq|k_b_tallt|k_b_xr|k_b_pupdate|k_b_rho" -c 12 \
  -o gpurun_out/prof_full -f python tools/profile_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
