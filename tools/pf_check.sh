# dev: sweep variant parity + wide-level probe
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep_cluster.py -x -q > gpurun_out/pf_test.log 2>&1; echo "rc=$?" >> gpurun_out/pf_test.log
for m in 0 2; do
  echo "== mode $m" >> gpurun_out/pf_probe.log
  RCG_SWEEP_CLUSTER=$m timeout 1200 python tools/config_probe.py c2 c4 c5 --mc --batch 0 >> gpurun_out/pf_probe.log 2>&1
done
