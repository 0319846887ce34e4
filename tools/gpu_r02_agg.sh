# Aggregate tensor with several chunks per thread (LCL_AGG_CH): parity, then cfg3 device round + kernel time.
O=gpurun_out/agg
mkdir -p $O
for p in 2 4; do
LCL_AGG_CH=$p timeout 900 python -m pytest tests -x -q -m gpu -k "aggregate or host_round or lclt" > $O/pytest_$p.log 2>&1; echo "pytest ch=$p rc=$?"; tail -1 $O/pytest_$p.log
done
for p in 1 2 4 1 2; do
  LCL_AGG_CH=$p timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --steps 5 > $O/b_$p.json 2> $O/b_$p.err
  python -c "
import json; d=json.load(open('$O/b_$p.json'))
k=[x for x in d['kernels'] if x['name']=='aggregate_tensor'][0]
print('ch=$p', round(d['value'],2), 'agg', round(k['ms'],3), 'ms', round(k['hbm_gbs']), 'GB/s')" || tail -3 $O/b_$p.err
done
