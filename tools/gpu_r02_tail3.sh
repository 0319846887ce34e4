# Host round: the last client's pairs accumulated slice by slice (LCL_LAST_PAIRS=1), cfg3.
O=gpurun_out/tail3
mkdir -p $O
for v in "5 1 1" "5 0 1" "12 1 1" "5 1 0" "5 1 1"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_LAST_PAIRS=$3 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$1_$2_$3.json 2> $O/e2e_$1_$2_$3.err
  python -c "import json; d=json.load(open('$O/e2e_$1_$2_$3.json')); print('cfg3 T=$1 prio=$2 lastpairs=$3', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$1_$2_$3.err
  grep -A20 "host round" $O/e2e_$1_$2_$3.err | tail -21 | grep "host round\|clients 1[789]"
done
