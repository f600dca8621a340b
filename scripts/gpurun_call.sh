# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
MET=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_summary; print(ncu_summary.EXTRA_METRICS)")
ncu --set full --metrics $MET --import-source on --clock-control none -k "regex:stn_|warp_|bslice_|det_" --launch-skip 13 --launch-count 13 -f -o gpurun_out/r2_step python scripts/prof_step.py 8 2 > gpurun_out/r2_step.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_step.ncu-rep gpurun_out/r2_ncu_step.md --traffic gpurun_out/ncu_traffic.json --pixels-per-launch 8388608 "stn_out_tile<0=stn_fwd" "stn_tables|stn_classify|stn_bwd_lean|stn_out_tile<1|stn_dx_scatter|stn_dtheta=stn_bwd" "warp_fwd=warp_fwd" "warp_bwd=warp_bwd" "bslice_fwd=bslice_fwd" "bslice_bwd|bslice_bounds|bslice_dgrid=bslice_bwd" >> gpurun_out/r2_step.log 2>&1
rm -f gpurun_out/r2_step.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-paper-shapes --no-cpu --no-e2e --no-next > gpurun_out/r2_launch_bench.log 2>&1
python scripts/launch_shares.py gpurun_out/r2_launches.csv > gpurun_out/r2_launch_shares.md 2>&1
tail -3 gpurun_out/r2_launch_shares.md
