# Resume check after the container was re-created: GPU suite, smoke, default bench.
O=gpurun_out/resume
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -n 2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1200 python bench.py --no-cpu > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python -c "import json; d=json.load(open('$O/bench_cfg3.json')); print('cfg3', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])" || tail -5 $O/bench_cfg3.err
