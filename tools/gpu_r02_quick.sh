# quick check after a kernel change: parity subset (or full with FULL=1), cfg3 bench breakdown
mkdir -p gpurun_out
if [ "${FULL:-0}" = 1 ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 900 python -m pytest tests -x -q -m gpu -k "evaluator or fused_hoisted or distance_matrix_bit_exact or hoisted or ntt or rescale or relin" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
tail -n 2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('round', round(d['value'],2)); [print(k['name'], k['launches'], round(k['ms'],3), round(k['hbm_gbs'])) for k in d['kernels']]" || tail -5 gpurun_out/bench_q.err
