# dev: round-2 final check -- bench first (the final line), ncu full of the batched sweeps only,
# then the whole GPU suite
mkdir -p gpurun_out /tmp/ncu
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?" >> gpurun_out/bench_final.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_b_sweepc|k_b_rho" -c 6 \
  -o /tmp/ncu/prof_sw -f python tools/profile_batched.py c3 24 2 deflation > gpurun_out/ncu_sw.log 2>&1
ncu -i /tmp/ncu/prof_sw.ncu-rep --page raw --csv > gpurun_out/prof_sw_raw.csv 2>/dev/null
timeout 2400 python -X faulthandler -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gt_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
