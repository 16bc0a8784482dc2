# dev: sweep variant parity (incl. per-level launches) + wide-level probe default vs grid
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep_cluster.py -x -q > gpurun_out/lv_test.log 2>&1; echo "rc=$?" >> gpurun_out/lv_test.log
for m in 2; do
  echo "== mode $m" >> gpurun_out/lv_probe.log
  RCG_SWEEP_CLUSTER=$m timeout 1200 python tools/config_probe.py c4 c5 c2 c3 --mc --batch 0 >> gpurun_out/lv_probe.log 2>&1
done
