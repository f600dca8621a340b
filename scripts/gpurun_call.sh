mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or graph" > gpurun_out/pytest_stn.log 2>&1; tail -1 gpurun_out/pytest_stn.log
python scripts/bench_layer.py 64 10 stn_bwd; python scripts/bench_paper.py stn
