mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for cfg in cfg2 cfg3; do for ln in ${LANES:-1 2 3}; do
  LCL_LANES=$ln timeout 600 python bench.py --config $cfg --no-cpu --steps 5 > gpurun_out/l_${cfg}_$ln.json 2> gpurun_out/l_${cfg}_$ln.err
  python -c "import json; d=json.load(open('gpurun_out/l_${cfg}_$ln.json')); print('$cfg lanes $ln', round(d['value'],3), 'e2e', round(d['e2e']['value'],2))" || tail -3 gpurun_out/l_${cfg}_$ln.err
done; done
