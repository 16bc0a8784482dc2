# dev: ncu --set full captures of the C3 bench kernels (batched at RT 24 with the deflation basis;
# single-RHS sweeps and SpMV) -> gpurun_out/prof_c3b.ncu-rep, prof_c3s.ncu-rep
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_b_sweepc|k_b_spmv_pq|k_b_tallt|k_b_deflate|k_b_pupdate|k_b_xr|k_b_rho" -c 14 \
  -o gpurun_out/prof_c3b -f python tools/profile_batched.py c3 24 2 deflation > gpurun_out/ncu_c3b.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_spmv" -c 6 \
  -o gpurun_out/prof_c3s -f python tools/sweep_tune.py c3 1 > gpurun_out/ncu_c3s.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3s.log
