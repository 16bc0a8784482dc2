# dev: cluster sweep phase counters (RCG_CL_PROF=1; =3 replaces DSMEM loads by local ones: timing only)
mkdir -p gpurun_out
for c in c1 c2; do for p in 1 3; do
  echo "== $c prof=$p" >> gpurun_out/cl_prof.log
  RCG_CL_PROF=$p RCG_SWEEP_CLUSTER=1 timeout 300 python tools/sweep_tune.py $c 20 >> gpurun_out/cl_prof.log 2>&1
done; done
