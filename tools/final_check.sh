# dev: the whole GPU suite + smoke + the default bench (logs under gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
