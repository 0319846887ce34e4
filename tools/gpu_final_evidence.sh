# End-of-round evidence: tests, smoke, bench (cfg2 with the CPU reference,
# cfg3), the reference arm, ncu launch list + per-kernel DRAM traffic,
# --set full of the ladder's column pass and ModUp/inner-product kernels,
# HE sweep, client-side timings.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg3 --no-cpu --steps 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
export LCL_LANES=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/one_round.py --config cfg2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/one_round.py --config cfg3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ntt_col_inv_lift_fwd|modup_ip_blk" --launch-skip 4 -c 2 -o gpurun_out/top_cfg2 python tools/one_round.py --config cfg2 > gpurun_out/ncu_top.log 2>&1
unset LCL_LANES
timeout 1500 python tools/he_sweep.py > gpurun_out/he_sweep.json 2> gpurun_out/he_sweep.err
timeout 900 python tools/client_encrypt_bench.py > gpurun_out/client_enc.json 2> gpurun_out/client_enc.err
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
