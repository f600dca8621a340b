mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "split_vs_tiled" 2>&1 | tail -1
