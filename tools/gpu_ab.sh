# A/B of library variants (paper_2408_06197_b200/_lib/variants/*.so) on the cfg3 round:
#   bash tools/gpu_ab.sh [bench args...]
mkdir -p gpurun_out/ab
for v in main $(cd paper_2408_06197_b200/_lib/variants && ls *.so | sed 's/\.so$//'); do
  if [ "$v" = main ]; then unset LCL_LIB_PATH; else export LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/$v.so; fi
  timeout 600 python bench.py --no-cpu --no-e2e --steps 10 "$@" > gpurun_out/ab/$v.json 2> gpurun_out/ab/$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab/$v.json')); print('$v', round(d['value'],2), [(x['name'], round(x['ms'],2)) for x in d['kernels'][:9]])" || tail -3 gpurun_out/ab/$v.err
done
unset LCL_LIB_PATH
