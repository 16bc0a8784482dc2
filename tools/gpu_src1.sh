mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_b_sweepc" -c 2 \
  -o /tmp/ncu/src1 -f python tools/profile_batched.py c3 24 1 none > gpurun_out/src1.log 2>&1
echo "rc=$?" >> gpurun_out/src1.log
ncu -i /tmp/ncu/src1.ncu-rep --page source --csv --print-source sass > gpurun_out/src1_sass.csv 2>/dev/null
ncu -i /tmp/ncu/src1.ncu-rep --page source --csv --print-source cuda > gpurun_out/src1_cuda.csv 2>/dev/null
ncu -i /tmp/ncu/src1.ncu-rep --page details --csv > gpurun_out/src1_details.csv 2>/dev/null
ls -la gpurun_out >> gpurun_out/src1.log
