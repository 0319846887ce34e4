mkdir -p gpurun_out
export LCL_LANES=1
LCL_COL_VARIANT=3 timeout 900 python -m pytest tests -x -q -m gpu -k "ntt or evaluator or bit_exact" 2>&1 | tail -2
for v in 0 1 2 3; do for c in cfg2 cfg3; do
  LCL_COL_VARIANT=$v timeout 600 python bench.py --config $c --no-cpu --steps 3 > gpurun_out/cv_${v}_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/cv_${v}_$c.json')); print('variant $v $c', round(d['value'],3), [(k['name'], round(k['ms'],3)) for k in d['kernels'] if k['name'].startswith('ntt_col')])"
done; done
