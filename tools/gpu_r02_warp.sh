# Pair CTAs sized to the schedule (one warp for <= 32 pairs): parity, e2e timeline.
O=gpurun_out/warp
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for t in 32 64 32; do
  LCL_PAIR_MIN_THREADS=$t LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_$t.json 2> $O/e2e_$t.err
  python -c "import json; d=json.load(open('$O/e2e_$t.json')); print('cfg3 min_threads=$t', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_$t.err
  grep -A20 "host round" $O/e2e_$t.err | tail -21 | grep "host round\|clients 1[6789]"
done
timeout 900 python bench.py --config cfg2 --no-cpu --steps 5 > $O/e2e2.json 2> $O/e2e2.err
python -c "import json; d=json.load(open('$O/e2e2.json')); print('cfg2', round(d['value'],2), round(d['e2e']['value'],2))"
