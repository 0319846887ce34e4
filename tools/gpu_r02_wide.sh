# Whole-matrix pair kernel on a 16-slot tile with 2 x 192 threads (LCL_PAIR_WIDE=2): parity, device round.
O=gpurun_out/wide
mkdir -p $O
LCL_PAIR_WIDE=2 timeout 1200 python -m pytest tests -x -q -m gpu -k "pair or distance or cfg3_benchmark or host_round" > $O/pytest.log 2>&1; echo "pytest wide rc=$?"; tail -1 $O/pytest.log
for v in 0 2 0 2; do
  LCL_PAIR_WIDE=$v timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --steps 5 > $O/b_$v.json 2> $O/b_$v.err
  python -c "
import json; d=json.load(open('$O/b_$v.json'))
k=[x for x in d['kernels'] if x['name']=='pair_accumulate'][0]
print('cfg3 wide=$v', round(d['value'],2), 'pair', round(k['ms'],2))" || tail -3 $O/b_$v.err
done
for v in 0 2; do
  LCL_PAIR_WIDE=$v timeout 900 python bench.py --config cfg2 --no-cpu --no-e2e --steps 5 > $O/b2_$v.json 2> $O/b2_$v.err
  python -c "
import json; d=json.load(open('$O/b2_$v.json'))
k=[x for x in d['kernels'] if x['name']=='pair_accumulate'][0]
print('cfg2 wide=$v', round(d['value'],3), 'pair', round(k['ms'],3))" || tail -3 $O/b2_$v.err
done
