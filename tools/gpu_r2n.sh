# dev: round-2 lines of the other BASELINE configurations (C1, C2, C5 with their reference arms) and C4 on one GPU
mkdir -p gpurun_out
CONFIGS="c1 c2 c5" bash tools/all_configs.sh
timeout 1200 python tools/c4_run.py > gpurun_out/c4_single_gpu.json 2> gpurun_out/c4_single_gpu.err; echo "c4 rc=$?" >> gpurun_out/all_configs.log
# dev A/B: the backward 16-byte-chunk sweep compiled for 8 (default) / 6 / 5 resident CTAs per SM
# (the 8-CTA build spills 16 bytes; alt libraries built by hand with -DRCG_BSWEEPC_BWD_MINB)
run() { echo "== $*" >> gpurun_out/ab_minb.log; env "$@" >> gpurun_out/ab_minb.log 2>&1; }
run A=default timeout 600 python tools/profile_batched.py c3 24 20 deflation
for mb in 6 5; do
  run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/alt/librcg_minb$mb.so timeout 600 python tools/profile_batched.py c3 24 20 deflation
  run RCG_LIB_PATH=$PWD/paper_2203_08498_b200/alt/librcg_minb$mb.so timeout 600 python tools/profile_batched.py c2 12 20 sc
done
run A=default timeout 600 python tools/profile_batched.py c2 12 20 sc
