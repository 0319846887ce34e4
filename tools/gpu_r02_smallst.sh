# Small pair sets (host-round single-client lanes) with a deeper copy ring (LCL_PAIR_SMALL_ST).
O=gpurun_out/smallst
mkdir -p $O
for st in 10 14; do
LCL_PAIR_SMALL_ST=$st timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or pair" > $O/pytest_$st.log 2>&1; echo "pytest st=$st rc=$?"; tail -1 $O/pytest_$st.log
done
for st in 0 10 14 10; do
  LCL_PAIR_SMALL_ST=$st LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$st.json 2> $O/e2e_$st.err
  python -c "import json; d=json.load(open('$O/e2e_$st.json')); print('cfg3 small_st=$st', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$st.err
  grep -A20 "host round" $O/e2e_$st.err | tail -21 | grep "host round\|clients 1[6789]"
done
LCL_PAIR_SMALL_ST=10 timeout 900 python bench.py --config cfg2 --no-cpu --steps 5 > $O/e2e2.json 2> $O/e2e2.err
python -c "import json; d=json.load(open('$O/e2e2.json')); print('cfg2 small_st=10', round(d['value'],2), round(d['e2e']['value'],2))"
