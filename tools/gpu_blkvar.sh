mkdir -p gpurun_out
export LCL_LANES=1
LCL_BLK_VARIANT=7 timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for v in ${BLKV:-0 1 2 4 7}; do for c in cfg2 cfg3; do
  LCL_BLK_VARIANT=$v timeout 600 python bench.py --config $c --no-cpu --steps 3 > gpurun_out/bv_${v}_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bv_${v}_$c.json')); print('variant $v $c', round(d['value'],3), [(k['name'], round(k['ms'],3)) for k in d['kernels'] if k['name'].startswith('ntt_blk') or k['name'].startswith('modup')])"
done; done
