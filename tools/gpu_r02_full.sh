# round 2 evidence: whole GPU suite, smoke, default bench (cfg3 + cpu_baseline),
# reference arm, cfg2 context line, traffic capture of one cfg3 round
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 8 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('ours', round(d['value'],2), d['e2e'], d['plan']['k'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline'])" || tail -5 gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_cfg3_ref.json 2> gpurun_out/bench_cfg3_ref.err
head -c 600 gpurun_out/bench_cfg3_ref.json; echo
timeout 600 python bench.py --config cfg2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg2.json')); print('cfg2', round(d['value'],2), d['e2e']['value'], d['cpu_baseline']['value'])" || tail -5 gpurun_out/bench_cfg2.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file /tmp/traffic_cfg3.csv python tools/one_round.py --config cfg3 --k 3 > /tmp/traffic.log 2>&1; echo "traffic rc=$?"
python tools/ncu_traffic.py /tmp/traffic_cfg3.csv > gpurun_out/r02_traffic_cfg3.json; head -c 400 gpurun_out/r02_traffic_cfg3.json
