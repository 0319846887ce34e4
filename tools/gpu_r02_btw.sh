# block-ordered twiddles: full GPU suite, cfg3 bench, ncu of the key-switch kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_btw.json 2> gpurun_out/bench_btw.err
python -c "import json; d=json.load(open('gpurun_out/bench_btw.json')); print('round', round(d['value'],2)); [print(k['name'], k['launches'], round(k['ms'],3), round(k['hbm_gbs'])) for k in d['kernels']]" || tail -5 gpurun_out/bench_btw.err
timeout 900 ncu --set full --clock-control none -k "regex:modup_ip_blk|ntt_blk_fwd|ntt_blk_inv|ntt_col_inv_lift" --launch-skip 20 -c 6 -o /tmp/btw python tools/one_round.py --config cfg3 --k 3 > /tmp/btw_prof.log 2>&1; echo "prof rc=$?"
ncu -i /tmp/btw.ncu-rep --page raw --csv > gpurun_out/r02_ncu_raw_btw.csv 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_raw_btw.csv > gpurun_out/r02_ncu_btw_summary.txt 2>&1; cat gpurun_out/r02_ncu_btw_summary.txt | head -40
