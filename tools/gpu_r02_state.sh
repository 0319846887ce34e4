# round 2 re-entry: GPU suite, smoke, default bench (cfg3), launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('ours', round(d['value'],2), d['e2e'], d['plan']['k'], d['roofline']['kernel'], d['roofline']['frac']); [print(k['name'], k['launches'], k['ms'], round(k['hbm_gbs'])) for k in d['kernels']]" || tail -5 gpurun_out/bench_cfg3.err
