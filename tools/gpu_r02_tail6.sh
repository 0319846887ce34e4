# Host round: small-pair-count accumulation variants (LCL_PAIR_SMALL_TE) with tail singles.
O=gpurun_out/tail6
mkdir -p $O
for te in 2 4; do
LCL_PAIR_SMALL_TE=$te LCL_TAIL_SINGLES=2 LCL_LANE_PRIO=1 LCL_LAST_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round or pair" > $O/pytest_$te.log 2>&1; echo "pytest te=$te rc=$?"; tail -1 $O/pytest_$te.log
done
for v in "5 1 0 2" "5 1 0 4" "5 1 1 2" "5 1 1 4" "5 0 0 2" "5 1 0 0"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_LAST_PAIRS=$3 LCL_PAIR_SMALL_TE=$4 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$1_$2_$3_$4.json 2> $O/e2e_$1_$2_$3_$4.err
  python -c "import json; d=json.load(open('$O/e2e_$1_$2_$3_$4.json')); print('cfg3 T=$1 prio=$2 lastpairs=$3 smallte=$4', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$1_$2_$3_$4.err
  grep -A20 "host round" $O/e2e_$1_$2_$3_$4.err | tail -21 | grep "host round\|clients 1[6789]"
done
