# parity tests, then bench per pair_accumulate / aggregate variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
for v in ${PA_VARIANTS:-0 10 11 12}; do
  LCL_PA_VARIANT=$v timeout 600 python bench.py --config ${CFG:-cfg3} --no-cpu --steps 3 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json; d=json.load(open('gpurun_out/var_$v.json')); print('variant $v', round(d['value'],3), [(k['name'], round(k['ms'],3)) for k in d['kernels'] if k['name'] in ('pair_accumulate','aggregate_tensor')])" || tail -3 gpurun_out/var_$v.err
done
