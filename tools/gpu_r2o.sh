# dev: bench --gpus 2 over the host-staged transport (two processes on the one GPU) with one
# allreduce per dot (RCG_DIST_FUSE=0) and with the fused reductions -- the collective count's
# effect where a collective is expensive (stream sync + gloo); NOT an NVLink number
mkdir -p gpurun_out
for c in c1 c2; do for f in 0 1; do
  RCG_DIST_FUSE=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + f)) \
    bench.py --gpus 2 --config $c --slab-transport host --steps 2 --warmup 1 > gpurun_out/slabs2_${c}_fuse$f.json 2> gpurun_out/slabs2_${c}_fuse$f.err
  echo "$c fuse=$f rc=$?" >> gpurun_out/slabs2.log
done; done
