# Host-round timeline at cfg3 (LCL_TRACE_ROUND): when the last byte lands vs when the lanes / D2H finish.
O=gpurun_out/trace
mkdir -p $O
for G in 8; do
  LCL_HOST_ROUND=$G LCL_TRACE_ROUND=1 timeout 900 python bench.py --config cfg3 --no-cpu --steps 3 > $O/e2e_G$G.json 2> $O/e2e_G$G.err
  python -c "import json; d=json.load(open('$O/e2e_G$G.json')); print('G=$G', round(d['value'],2), round(d['e2e']['value'],2))" || tail -3 $O/e2e_G$G.err
  grep "host round" $O/e2e_G$G.err | tail -3
done
