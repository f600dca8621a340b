# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp or host" 2>&1 | tail -1
python scripts/collapse_margin.py 3 | grep -v scatter
python scripts/bench_warp.py
python scripts/bench_layer.py 64 10 warp_bwd
