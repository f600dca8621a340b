mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
