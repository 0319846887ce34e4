# round 2: the new paths first (fused hoisting, distance modes, pairwise
# entry, LCLT), then the whole GPU suite, the cfg3 bench and the HE sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "fused_hoisted or distance_modes or pairwise_distance_entry or lclt and not reference_bytes" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
tail -n 30 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -q -m gpu -k "not reference_bytes and not cfg3_benchmark" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 6 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('ours', round(d['value'],2), d['e2e']['value'], d['plan']['k'], d['roofline']['kernel'], d['roofline']['frac'], [(x['name'], round(x['ms'],2)) for x in d['kernels'][:10]])" || tail -5 gpurun_out/bench_cfg3.err
timeout 900 python tools/he_sweep.py --no-ref > gpurun_out/he_sweep.json 2> gpurun_out/he_sweep.err; tail -5 gpurun_out/he_sweep.err
