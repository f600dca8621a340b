# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
python scripts/collapse_margin.py 5 2>&1 | grep auto
RSGRAD_WARP_R=16 python scripts/collapse_margin.py 5 2>&1 | grep auto
RSGRAD_WARP_R=16 python scripts/bench_warp.py
python scripts/bench_warp.py
