# milestone check: full GPU suite, smoke, the default bench line (cfg3 + cpu_baseline + e2e)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('round', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks']); [print(k['name'], k['launches'], round(k['ms'],3), round(k['hbm_gbs'])) for k in d['kernels']]" || tail -5 gpurun_out/bench_cfg3.err
