# dev: round-2 lines of the other BASELINE configurations (C1, C2, C5 with their reference arms) and C4 on one GPU
mkdir -p gpurun_out
CONFIGS="c1 c2 c5" bash tools/all_configs.sh
timeout 1200 python tools/c4_run.py > gpurun_out/c4_single_gpu.json 2> gpurun_out/c4_single_gpu.err; echo "c4 rc=$?" >> gpurun_out/all_configs.log
