# source-level ncu of the column pass and modup_ip_blk (one launch each, cfg3)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:ntt_col_inv_lift_fwd|modup_ip_blk|ntt_blk_fwd" --launch-skip 24 -c 5 -o /tmp/src python tools/one_round.py --config cfg3 --k 3 > /tmp/src.log 2>&1; echo "prof rc=$?"
ncu -i /tmp/src.ncu-rep --page raw --csv > gpurun_out/r02_src_raw.csv 2>&1
for k in ntt_col_inv_lift_fwd modup_ip_blk ntt_blk_fwd; do
  ncu -i /tmp/src.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 --print-source sass > gpurun_out/r02_src_sass_$k.csv 2>&1
done
ls -la gpurun_out/r02_src*
