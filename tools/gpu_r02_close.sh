# Closing evidence after the host-round tail work: GPU suite, smoke, default bench
# (cfg3 + cpu_baseline + e2e), cfg2 line, reference arm.
O=gpurun_out/close
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -n 2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python -c "import json; d=json.load(open('$O/bench_cfg3.json')); print('cfg3', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])" || tail -5 $O/bench_cfg3.err
timeout 900 python bench.py --config cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "import json; d=json.load(open('$O/bench_cfg2.json')); print('cfg2', round(d['value'],3), 'e2e', round(d['e2e']['value'],2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']))" || tail -5 $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_cfg3_ref.json 2> $O/bench_cfg3_ref.err
python -c "import json; d=json.load(open('$O/bench_cfg3_ref.json')); print('ref', d.get('value'), d.get('cpu_baseline',{}).get('sample'))"
