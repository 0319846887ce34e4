# Pair kernel with W warps on a W*8-slot tile for <= 32 pairs (LCL_PAIR_W): full GPU suite, e2e timeline.
O=gpurun_out/w
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
LCL_PAIR_W=2 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or pair or distance" > $O/pytest_w2.log 2>&1; echo "pytest w2 rc=$?"; tail -1 $O/pytest_w2.log
for w in 4 1 2 4; do
  LCL_PAIR_W=$w LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$w.json 2> $O/e2e_$w.err
  python -c "import json; d=json.load(open('$O/e2e_$w.json')); print('cfg3 W=$w', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$w.err
  grep -A20 "host round" $O/e2e_$w.err | tail -21 | grep "host round\|clients 1[789]"
done
for w in 4 1; do
LCL_PAIR_W=$w timeout 900 python bench.py --config cfg2 --no-cpu --steps 5 > $O/e2e2_$w.json 2> $O/e2e2_$w.err
python -c "import json; d=json.load(open('$O/e2e2_$w.json')); print('cfg2 W=$w', round(d['value'],2), round(d['e2e']['value'],2))"
done
