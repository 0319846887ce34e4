# Runs bench.py's multi-rank path (chunk-sharded round, reduce_scatter /
# all-gather) as 2 and 3 ranks on ONE GPU over gloo: an orchestration smoke
# test for boxes with a single B200. Its timings are not N-GPU numbers.
mkdir -p gpurun_out
for w in 2 3; do
  LCL_DIST_BACKEND=gloo LCL_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node $w --master-addr 127.0.0.1 --master-port 29$((500 + w)) bench.py --gpus $w \
    --steps 2 --warmup 3 --no-cpu > gpurun_out/multirank_$w.json 2> gpurun_out/multirank_$w.err
  echo "world $w rc=$?"; tail -c 400 gpurun_out/multirank_$w.json; tail -3 gpurun_out/multirank_$w.err
done
