# Host round with CUDA_DEVICE_MAX_CONNECTIONS=32: trailing singles x priority, cfg3 and cfg2.
O=gpurun_out/tail2
mkdir -p $O
for v in "3 1" "5 1" "8 1" "8 0" "12 1"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$1_$2.json 2> $O/e2e_$1_$2.err
  python -c "import json; d=json.load(open('$O/e2e_$1_$2.json')); print('cfg3 T=$1 prio=$2', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$1_$2.err
  grep -A14 "host round" $O/e2e_$1_$2.err | tail -15 | grep -v "lane [0-4] "
done
for v in "0 0" "0 1" "2 1"; do
  set -- $v
  LCL_TAIL_SINGLES=$1 LCL_LANE_PRIO=$2 timeout 900 python bench.py --config cfg2 --no-cpu --steps 5 > $O/e2e2_$1_$2.json 2> $O/e2e2_$1_$2.err
  python -c "import json; d=json.load(open('$O/e2e2_$1_$2.json')); print('cfg2 T=$1 prio=$2', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e2_$1_$2.err
done
