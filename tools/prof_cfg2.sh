# ncu --set full of the first launches of every path kernel in one cfg2 round
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:ntt_|modup|pair_acc" -c 14 -o gpurun_out/prof_cfg2 python tools/one_round.py --config cfg2 > gpurun_out/prof_cfg2.log 2>&1
tail -n 3 gpurun_out/prof_cfg2.log
