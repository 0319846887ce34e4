# host-round parity, then e2e at cfg3 / cfg2: the aggregate finished in 4 pieces (main) vs 1 (ap1)
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -x -q -m gpu -k "host_round or lclt or server_round" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for v in main ap1; do
for cfg in cfg3 cfg2; do
  if [ $v = main ]; then unset LCL_LIB_PATH; else export LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/$v.so; fi
  timeout 900 python bench.py --config $cfg --no-cpu --steps 5 > gpurun_out/ab/e2e_${cfg}_$v.json 2> gpurun_out/ab/e2e_${cfg}_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab/e2e_${cfg}_$v.json')); print('$cfg $v', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 gpurun_out/ab/e2e_${cfg}_$v.err
done; done; done
unset LCL_LIB_PATH
