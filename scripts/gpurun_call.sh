mkdir -p gpurun_out
for r in 8 4; do echo "R=$r"; RSGRAD_WARP_R=$r python scripts/bench_paper.py warp; RSGRAD_WARP_R=$r python scripts/bench_layer.py 8 20 warp_bwd; RSGRAD_WARP_R=$r python scripts/bench_layer.py 64 10 warp_bwd; done
RSGRAD_WARP_R=4 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp and (collapse or parity or determin)" 2>&1 | tail -2
RSGRAD_WARP_R=4 python scripts/collapse_margin.py 5 2>&1 | tail -5
python scripts/collapse_margin.py 5 2>&1 | tail -5
