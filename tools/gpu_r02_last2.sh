# Sliced last group: per-lane timeline, and the last lane on a high-priority stream.
O=gpurun_out/last2
mkdir -p $O
LCL_LANE_PRIO=1 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for cfg in cfg3 cfg2; do
for v in "8 0" "8 1"; do
  set -- $v
  LCL_LAST_SLICES=$1 LCL_LANE_PRIO=$2 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config $cfg --no-cpu --steps 3 > $O/e2e_${cfg}_$1_$2.json 2> $O/e2e_${cfg}_$1_$2.err
  python -c "import json; d=json.load(open('$O/e2e_${cfg}_$1_$2.json')); print('$cfg S=$1 prio=$2', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_${cfg}_$1_$2.err
  grep -A8 "host round" $O/e2e_${cfg}_$1_$2.err | tail -9
done
done
