# parity tests + cfg2/cfg3 bench (FP64 rows on, then forced off for an A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
LCL_FP64=0 timeout 600 python bench.py --no-cpu > gpurun_out/bench_cfg2_int.json 2> gpurun_out/bench_cfg2_int.err
timeout 600 python bench.py --config cfg3 --no-cpu --steps 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for f in gpurun_out/bench_cfg2.json gpurun_out/bench_cfg2_int.json gpurun_out/bench_cfg3.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['e2e']['value'], [(k['name'], round(k['ms'],3)) for k in d['kernels']])" || tail -5 ${f%.json}.err; done
