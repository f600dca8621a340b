mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp or graph" > gpurun_out/pytest_w.log 2>&1; tail -1 gpurun_out/pytest_w.log
python scripts/bench_paper.py warp; python scripts/bench_layer.py 64 10 warp_bwd
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:det_scatter python scripts/bench_paper.py warp 2>/dev/null | grep det_scatter | head -3 | cut -c1-200
