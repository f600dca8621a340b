mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or warp or graph" 2>&1 | tail -1
python scripts/bench_paper.py stn; python scripts/bench_paper.py warp
