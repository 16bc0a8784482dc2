# dev: one GPU test file / selection (TESTS="..." K="...")
mkdir -p gpurun_out
timeout 1500 python -X faulthandler -m pytest $TESTS -x -q -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/one.log 2>&1; echo "rc=$?" >> gpurun_out/one.log
