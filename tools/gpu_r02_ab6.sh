# A/B: divide-and-round block pass with TMA-staged operands (main) vs register loads (drold); two slot_reduce lanes at cfg3
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -x -q -m gpu -k "evaluator or hoisted or distance_matrix_bit_exact or host_round or rescale or relin or cfg3" > gpurun_out/pytest_gpu.log 2>&1; echo "main pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
run() { timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab/$1.json 2> gpurun_out/ab/$1.err; python -c "import json; d=json.load(open('gpurun_out/ab/$1.json')); print('$1', round(d['value'],2), [(x['name'], round(x['ms'],2)) for x in d['kernels'][:9]])" || tail -3 gpurun_out/ab/$1.err; }
run tma
LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/drold.so run drold
LCL_LANES=2 run lanes2
run tma2
