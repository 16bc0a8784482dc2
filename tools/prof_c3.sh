# dev: ncu --set full captures of the C3 bench kernels (batched at RT 24 with the deflation basis;
# single-RHS sweeps and SpMV); only CSV summaries come back (the .ncu-rep stay on the box)
mkdir -p gpurun_out /tmp/ncu
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_b_sweepc|k_b_spmv_pq|k_b_tallt|k_b_deflate|k_b_pupdate|k_b_xr|k_b_rho" -c 14 \
  -o /tmp/ncu/prof_c3b -f python tools/profile_batched.py c3 24 2 deflation > gpurun_out/ncu_c3b.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_spmv" -c 6 \
  -o /tmp/ncu/prof_c3s -f python tools/sweep_tune.py c3 1 > gpurun_out/ncu_c3s.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3s.log
for r in prof_c3b prof_c3s; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
ls -la gpurun_out/*.csv >> gpurun_out/ncu_c3b.log
