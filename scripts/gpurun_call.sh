# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp" > gpurun_out/r2_pt_warp.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pt_warp.log
for i in 1 2 3 4 5; do timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "collapse_paper" 2>&1 | tail -1; done
python scripts/bench_warp.py
python scripts/bench_layer.py 64 10 warp_bwd
