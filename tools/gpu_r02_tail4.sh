# Host round: last two lanes high priority, last group's slice accumulations low priority.
O=gpurun_out/tail5
mkdir -p $O
LCL_TAIL_SINGLES=2 LCL_LANE_PRIO=1 LCL_LAST_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for v in "5 1 1" "3 1 1" "8 1 1" "5 1 0" "5 1 1"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_LAST_PAIRS=$3 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$1_$2_$3.json 2> $O/e2e_$1_$2_$3.err
  python -c "import json; d=json.load(open('$O/e2e_$1_$2_$3.json')); print('cfg3 T=$1 prio=$2 lastpairs=$3', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$1_$2_$3.err
  grep -A20 "host round" $O/e2e_$1_$2_$3.err | tail -21 | grep "host round\|clients 1[789]"
done
for v in "0 0 0" "0 1 1" "0 1 0"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_LAST_PAIRS=$3 timeout 900 python bench.py --config cfg2 --no-cpu --steps 5 > $O/e2e2_$1_$2_$3.json 2> $O/e2e2_$1_$2_$3.err
  python -c "import json; d=json.load(open('$O/e2e2_$1_$2_$3.json')); print('cfg2 T=$1 prio=$2 lastpairs=$3', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e2_$1_$2_$3.err
done
