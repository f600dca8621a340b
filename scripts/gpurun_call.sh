# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; tail -c 300 gpurun_out/bench_r2i.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_r2i.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/paper_r2i.csv python scripts/bench_paper.py --launches gpurun_out/paper_r2i.csv.order > gpurun_out/pl.log 2>&1
python scripts/bench_paper.py --parse gpurun_out/paper_r2i.csv > gpurun_out/paper_breakdown_r2i.md 2>&1
MET=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_summary; print(ncu_summary.EXTRA_METRICS)")
timeout 1200 ncu --set full --metrics $MET --import-source on --clock-control none -k "regex:stn_|warp_|bslice_|det_" --launch-skip 13 --launch-count 13 -f -o gpurun_out/r2i_step python scripts/prof_step.py 8 2 > gpurun_out/ncu_step.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2i_step.ncu-rep gpurun_out/r2i_ncu_step.md --traffic gpurun_out/ncu_traffic_r2i.json --pixels-per-launch 8388608 "stn_out_tile<0=stn_fwd" "stn_prep|stn_bwd_lean|stn_out_tile<1|stn_dx_scatter|stn_dtheta=stn_bwd" "warp_fwd=warp_fwd" "warp_bwd|det_scatter=warp_bwd" "bslice_fwd=bslice_fwd" "bslice_bounds|bslice_bwd|bslice_dgrid=bslice_bwd" >> gpurun_out/ncu_step.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
