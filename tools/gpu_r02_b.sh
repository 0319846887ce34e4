# round 2: LCLT / C++ mirror / cfg3 golden tests, cfg3 launch list + ncu of the key-switch kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -k "lclt or cpp_mirror or cfg3_benchmark or fused_hoisted" > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
tail -n 25 gpurun_out/pytest_b.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-graph > gpurun_out/launch_bench.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:modup_ip_hoist|modup_ip_blk|ntt_col_inv_lift|ntt_blk_fwd|ntt_blk_inv" -c 12 -o gpurun_out/r02_prof_cfg3 python tools/one_round.py --config cfg3 --k 3 > gpurun_out/prof_cfg3.log 2>&1; echo "prof rc=$?"
tail -n 3 gpurun_out/prof_cfg3.log
