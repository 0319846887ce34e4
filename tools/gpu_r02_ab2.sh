# A/B batch 2: register-prefetched ModUp digits (pf6/pf8), column pass with the
# source tile parked in shared memory (colv3) or at 2 CTAs/SM (col2); parity
# subset per variant, then the cfg3 bench of each.
mkdir -p gpurun_out
for v in $(cd paper_2408_06197_b200/_lib/variants && ls *.so | sed 's/\.so$//'); do
  LCL_LIB_PATH=$PWD/paper_2408_06197_b200/_lib/variants/$v.so timeout 900 python -m pytest tests -x -q -m gpu -k "evaluator or fused_hoisted or distance_matrix_bit_exact or hoisted" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -1 gpurun_out/pytest_$v.log
done
bash tools/gpu_ab.sh
