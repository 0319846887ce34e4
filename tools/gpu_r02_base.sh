# round-2 baseline: GPU parity suite + cfg3 at unfold factors 1..5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
for k in 1 2 3 4 5; do
  timeout 600 python bench.py --config cfg3 --no-cpu --no-e2e --steps 5 --k $k > gpurun_out/bench_cfg3_k$k.json 2> gpurun_out/bench_cfg3_k$k.err
  python -c "import json; d=json.load(open('gpurun_out/bench_cfg3_k$k.json')); print('k=$k', round(d['value'],2), [(x['name'], round(x['ms'],2)) for x in d['kernels'][:8]])" || tail -3 gpurun_out/bench_cfg3_k$k.err
done
