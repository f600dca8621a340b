ncu --set full --import-source on --clock-control none -k "regex:stn_|warp_|bslice_" --launch-skip 13 --launch-count 13 -f -o gpurun_out/step_v8 python scripts/prof_step.py 8 2 > gpurun_out/step_v8.log 2>&1; echo ncufull=$?
python scripts/ncu_summary.py gpurun_out/step_v8.ncu-rep gpurun_out/step_v8.md --traffic gpurun_out/ncu_traffic.json --pixels-per-launch 8388608 \
  "stn_bwd_lean|stn_classify|stn_tables|stn_dtheta_finalize|stn_dx_scatter|stn_out_tile<1=stn_bwd" "stn_out_tile<0=stn_fwd" \
  "warp_fwd=warp_fwd" "warp_bwd=warp_bwd" "bslice_fwd=bslice_fwd" "bslice_bwd|bslice_dgrid|bslice_bounds=bslice_bwd" >> gpurun_out/step_v8.log 2>&1
for k in stn_bwd_lean stn_out_tile bslice_bwd_tiled warp_bwd_kernel; do
  ncu -i gpurun_out/step_v8.ncu-rep --page source --csv --print-source cuda,sass -k "regex:$k" > /tmp/src_$k.csv 2>/dev/null
  echo "=== $k" >> gpurun_out/step_v8.hot.txt; python scripts/src_hot.py /tmp/src_$k.csv 40 >> gpurun_out/step_v8.hot.txt 2>&1
done
rm -f gpurun_out/step_v8.ncu-rep
cut -c1-300 gpurun_out/step_v8.md; cat gpurun_out/ncu_traffic.json | head -12
