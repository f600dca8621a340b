mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp" > gpurun_out/pytest_w.log 2>&1; tail -2 gpurun_out/pytest_w.log
for nb in 8 16 32 64; do echo nb=$nb; python scripts/bench_layer.py $nb 20 warp_fwd; RSGRAD_WARP_FWD_G=1 python scripts/bench_layer.py $nb 20 warp_fwd; done
python scripts/bench_paper.py warp
