# Sliced last group in the host round: parity, then e2e at cfg3 / cfg2 per slice count.
O=gpurun_out/last
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
LCL_LAST_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > $O/pytest_pairs.log 2>&1; echo "pytest pairs rc=$?"; tail -1 $O/pytest_pairs.log
for cfg in cfg3 cfg2; do
for v in "1 0" "8 0" "8 1" "4 1" "16 1"; do
  set -- $v
  LCL_LAST_SLICES=$1 LCL_LAST_PAIRS=$2 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config $cfg --no-cpu --steps 3 > $O/e2e_${cfg}_$1_$2.json 2> $O/e2e_${cfg}_$1_$2.err
  python -c "import json; d=json.load(open('$O/e2e_${cfg}_$1_$2.json')); print('$cfg S=$1 pairs=$2', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_${cfg}_$1_$2.err
  grep "host round" $O/e2e_${cfg}_$1_$2.err | tail -1
done
done
