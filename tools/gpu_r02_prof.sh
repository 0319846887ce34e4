# round 2: new KGC tests, cfg3 launch list (summarised on the box) and ncu --set full of the key-switch kernels (exported to CSV, report dropped)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "kgc_distance_table or lclt" > gpurun_out/pytest_c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c.log
tail -n 5 gpurun_out/pytest_c.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-graph > /tmp/launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py /tmp/launches.csv > gpurun_out/r02_launches_cfg3_summary.txt 2>&1; head -30 gpurun_out/r02_launches_cfg3_summary.txt
gzip -c /tmp/launches.csv > gpurun_out/r02_launches_cfg3.csv.gz; ls -la gpurun_out/
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:modup_ip_hoist|modup_ip_blk|ntt_col_inv_lift|ntt_blk_fwd|ntt_blk_inv" -c 12 -o /tmp/r02_prof_cfg3 python tools/one_round.py --config cfg3 --k 3 > /tmp/prof_cfg3.log 2>&1; echo "prof rc=$?"
ncu -i /tmp/r02_prof_cfg3.ncu-rep --page raw --csv > gpurun_out/r02_ncu_raw_cfg3.csv 2>&1
ncu -i /tmp/r02_prof_cfg3.ncu-rep --page details --csv > gpurun_out/r02_ncu_details_cfg3.csv 2>&1
ncu -i /tmp/r02_prof_cfg3.ncu-rep --page source --csv --kernel-name regex:modup_ip_hoist > gpurun_out/r02_ncu_source_hoist.csv 2>&1
ls -la gpurun_out/
