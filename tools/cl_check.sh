# dev: cluster sweep -- parity tests first (bounded), then sweep timings grid vs cluster variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep_cluster.py -x -q > gpurun_out/cl_test.log 2>&1; echo "rc=$?" >> gpurun_out/cl_test.log
for c in c1 c2; do
  echo "== $c grid" >> gpurun_out/cl_tune.log; RCG_SWEEP_CLUSTER=0 timeout 300 python tools/sweep_tune.py $c 20 >> gpurun_out/cl_tune.log 2>&1
  echo "== $c cluster 227" >> gpurun_out/cl_tune.log; RCG_SWEEP_CLUSTER=1 timeout 300 python tools/sweep_tune.py $c 20 >> gpurun_out/cl_tune.log 2>&1
  echo "== $c cluster 100KB carve50" >> gpurun_out/cl_tune.log; RCG_CL_SMEM_KB=100 RCG_CL_CARVEOUT=50 RCG_SWEEP_CLUSTER=1 timeout 300 python tools/sweep_tune.py $c 20 >> gpurun_out/cl_tune.log 2>&1
  echo "== $c cluster all carve100" >> gpurun_out/cl_tune.log; RCG_CARVEOUT=100 RCG_CL_CARVEOUT=100 RCG_SWEEP_CLUSTER=1 timeout 300 python tools/sweep_tune.py $c 20 >> gpurun_out/cl_tune.log 2>&1
done
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --no-variants > gpurun_out/bench_cl.json 2> gpurun_out/bench_cl.err
fi
