# Multi-rank orchestration on ONE B200 (gloo, LCL_ONE_DEVICE): bench.py's chunk-sharded
# round as 2 and 3 ranks (torchrun) at cfg3, and the --gpus 2 self-launch at cfg2.
# Timings are not N-GPU numbers; this checks the sharded path end to end on the device.
mkdir -p gpurun_out
for w in 2 3; do
  LCL_DIST_BACKEND=gloo LCL_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node $w --master-addr 127.0.0.1 --master-port 29$((500 + w)) bench.py --gpus $w \
    --steps 2 --warmup 3 --no-cpu > gpurun_out/multirank_$w.json 2> gpurun_out/multirank_$w.err
  echo "world $w rc=$?"; python -c "import json; d=json.load(open('gpurun_out/multirank_$w.json')); print(d['n_gpus'], round(d['value'],2), d.get('scaling'), d['config'].get('parallelism', d.get('parallelism')))" || tail -3 gpurun_out/multirank_$w.err
done
LCL_DIST_BACKEND=gloo LCL_ONE_DEVICE=1 timeout 900 python bench.py --gpus 2 --config cfg2 --steps 2 --warmup 3 --no-cpu > gpurun_out/selflaunch_2.json 2> gpurun_out/selflaunch_2.err
echo "self-launch rc=$?"; python -c "import json; d=json.load(open('gpurun_out/selflaunch_2.json')); print(d['n_gpus'], round(d['value'],2))" || tail -3 gpurun_out/selflaunch_2.err
timeout 600 python -m pytest tests -q -m gpu -k "shard" > gpurun_out/pytest_shard.log 2>&1; echo "shard tests rc=$?"; tail -1 gpurun_out/pytest_shard.log
