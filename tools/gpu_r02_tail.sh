# Host round: trailing single-client groups (LCL_TAIL_SINGLES) x last-lane priority, cfg3.
O=gpurun_out/tail
mkdir -p $O
LCL_TAIL_SINGLES=2 LCL_LANE_PRIO=1 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for v in "0 0" "3 0" "5 0" "5 1" "8 1" "5 1"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$1_$2.json 2> $O/e2e_$1_$2.err
  python -c "import json; d=json.load(open('$O/e2e_$1_$2.json')); print('cfg3 T=$1 prio=$2', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$1_$2.err
  grep -A14 "host round" $O/e2e_$1_$2.err | tail -15
done
