# Final round-2 evidence on the closing code: smoke, default bench (cfg3 + cpu_baseline + e2e), cfg2, cfg4 device.
O=gpurun_out/final4
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python -c "import json; d=json.load(open('$O/bench_cfg3.json')); print('cfg3', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'], d['gpu_launches'])" || tail -5 $O/bench_cfg3.err
timeout 900 python bench.py --config cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "import json; d=json.load(open('$O/bench_cfg2.json')); print('cfg2', round(d['value'],3), 'e2e', round(d['e2e']['value'],2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']))" || tail -5 $O/bench_cfg2.err
timeout 900 python bench.py --config cfg4 --no-e2e --no-cpu --steps 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python -c "import json; d=json.load(open('$O/bench_cfg4.json')); print('cfg4', round(d['value'],2))" || tail -5 $O/bench_cfg4.err
