# Round-2 evidence: GPU suite, smoke, default bench (cfg3 + cpu_baseline + e2e),
# reference arm, cfg2 and cfg4 lines, ncu traffic + launch list of cfg3, ncu
# --set full of the top kernels, HE sweep.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -n 2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python -c "import json; d=json.load(open('$O/bench_cfg3.json')); print('cfg3', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), d['roofline'])" || tail -5 $O/bench_cfg3.err
timeout 900 python bench.py --impl reference > $O/bench_cfg3_ref.json 2> $O/bench_cfg3_ref.err
head -c 400 $O/bench_cfg3_ref.json; echo
timeout 900 python bench.py --config cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "import json; d=json.load(open('$O/bench_cfg2.json')); print('cfg2', round(d['value'],3), 'e2e', round(d['e2e']['value'],2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']))" || tail -5 $O/bench_cfg2.err
timeout 1200 python bench.py --config cfg4 --no-cpu --no-e2e --steps 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python -c "import json; d=json.load(open('$O/bench_cfg4.json')); print('cfg4', round(d['value'],2))" || tail -5 $O/bench_cfg4.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file /tmp/traffic_cfg3.csv python tools/one_round.py --config cfg3 --k 3 > /tmp/traffic.log 2>&1; echo "traffic rc=$?"
python tools/ncu_traffic.py /tmp/traffic_cfg3.csv > $O/r02_traffic_cfg3.json; head -c 300 $O/r02_traffic_cfg3.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > /tmp/launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py /tmp/launches.csv > $O/r02_launches_cfg3_summary.txt 2>&1; head -14 $O/r02_launches_cfg3_summary.txt
gzip -c /tmp/launches.csv > $O/r02_launches_cfg3.csv.gz
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:pair_accumulate|modup_ip_blk|ntt_col_inv_lift|ntt_blk_fwd|aggregate_stream|ntt_blk_inv" --launch-skip 20 -c 7 -o /tmp/final python tools/one_round.py --config cfg3 --k 3 > /tmp/final_prof.log 2>&1; echo "prof rc=$?"
ncu -i /tmp/final.ncu-rep --page raw --csv > $O/r02_ncu_raw_final.csv 2>&1
python tools/ncu_summary.py $O/r02_ncu_raw_final.csv > $O/r02_ncu_full_final.txt 2>&1; grep "==" $O/r02_ncu_full_final.txt
timeout 1500 python tools/he_sweep.py > $O/he_sweep.json 2> $O/he_sweep.err; echo "sweep rc=$?"
ls -la $O
