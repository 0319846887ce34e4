mkdir -p gpurun_out
for v in keys2 keys1; do
  LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/$v.so timeout 900 python -m pytest tests -x -q -m gpu -k "evaluator or fused_hoisted or distance_matrix_bit_exact or server_round_concurrent" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -2 gpurun_out/pytest_$v.log
done
bash tools/gpu_ab.sh
