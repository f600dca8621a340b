mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or graph" > gpurun_out/pytest_stn.log 2>&1; tail -2 gpurun_out/pytest_stn.log
python scripts/bench_layer.py 64 10 stn_bwd; python scripts/bench_paper.py stn; RSGRAD_STN_PREP=1 python scripts/bench_paper.py stn
