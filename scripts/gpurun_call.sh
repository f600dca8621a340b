mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp" > gpurun_out/pytest_w.log 2>&1; tail -2 gpurun_out/pytest_w.log
python scripts/bench_layer.py 64 20 warp_bwd
python scripts/bench_paper.py warp
