# Round evidence on one B200: parity tests, smoke, default bench (cfg2, with the
# CPU reference baseline), cfg3 bench, ncu launch list + per-kernel DRAM
# traffic of one cfg2 round, ncu --set full of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg3 --no-cpu --steps 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/one_round.py --config cfg2 > gpurun_out/ncu_traffic.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${TOPK:-modup_ip_blk}" -c 1 -o gpurun_out/top_cfg2 python tools/one_round.py --config cfg2 > gpurun_out/ncu_top.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
