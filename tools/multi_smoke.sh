# run bench.py's N>1 path on a single-GPU box: ranks share the GPU, gloo transport
for N in 2 4; do
LOD_DIST_BACKEND=gloo LOD_POOL_RESERVE_MIB=1024 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 6 --warmup 3 --arena-gib 4 \
  > gpurun_out/multi_$N.json 2> gpurun_out/multi_$N.err
echo "N=$N rc=$?"; tail -c 1200 gpurun_out/multi_$N.json; grep -iE "error|Traceback" gpurun_out/multi_$N.err | head -5
done
