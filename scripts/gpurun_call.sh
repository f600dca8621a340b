# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp" 2>&1 | tail -2
