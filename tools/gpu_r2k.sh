# dev: round-2 re-entry -- the whole GPU suite (parity records come back under gpurun_out/parity)
mkdir -p gpurun_out
timeout 2400 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
