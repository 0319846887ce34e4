# round 2: GPU parity suite, then the default bench (cfg3, dynamic hoisting,
# cpu_baseline on the host) and the reference arm on the same box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
nproc
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('ours', round(d['value'],2), d['e2e']['value'], d['plan'], d['cpu_baseline'], d['roofline'])" || tail -5 gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_cfg3_ref.json 2> gpurun_out/bench_cfg3_ref.err
cat gpurun_out/bench_cfg3_ref.json | head -c 1500; tail -3 gpurun_out/bench_cfg3_ref.err
