# host-round parity, then e2e at cfg3 / cfg2 with the round's timeline (aggregate D2H on its own stream)
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for cfg in cfg3 cfg2; do
  LCL_TRACE_ROUND=1 timeout 900 python bench.py --config $cfg --no-cpu --steps 5 > gpurun_out/ab/e2e_${cfg}.json 2> gpurun_out/ab/e2e_${cfg}.err
  python -c "import json; d=json.load(open('gpurun_out/ab/e2e_${cfg}.json')); print('$cfg', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 gpurun_out/ab/e2e_${cfg}.err
  grep "host round" gpurun_out/ab/e2e_${cfg}.err | tail -2
done
