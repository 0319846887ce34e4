mkdir -p gpurun_out
for v in ${PV:-10}; do
LCL_PA_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pair_acc" -c 1 -o gpurun_out/prof_paf_$v python tools/one_round.py --config cfg3 > gpurun_out/prof_paf_$v.log 2>&1
tail -2 gpurun_out/prof_paf_$v.log
done
