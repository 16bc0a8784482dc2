# dev: the whole GPU suite without -x (bounded), durations, parity log
mkdir -p gpurun_out
timeout 3000 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 -o faulthandler_timeout=900 > gpurun_out/gt_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gt_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
