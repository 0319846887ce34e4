# A/B: single rotations through modup_ip_hoist (rh) vs modup_ip_blk (main)
mkdir -p gpurun_out/ab
LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/rh.so timeout 900 python -m pytest tests -x -q -m gpu -k "evaluator or hoisted or distance_matrix_bit_exact or cfg3 or rotate" > gpurun_out/pytest_rh.log 2>&1; echo "rh pytest rc=$?"; tail -1 gpurun_out/pytest_rh.log
run() { timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab/$1.json 2> gpurun_out/ab/$1.err; python -c "import json; d=json.load(open('gpurun_out/ab/$1.json')); print('$1', round(d['value'],2), [(x['name'], round(x['ms'],2)) for x in d['kernels'][:9]])" || tail -3 gpurun_out/ab/$1.err; }
run main
LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/rh.so run rh
