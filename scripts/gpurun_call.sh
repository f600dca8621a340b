mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bslice" > gpurun_out/pytest_bs.log 2>&1; tail -2 gpurun_out/pytest_bs.log
python scripts/bench_paper.py bslice; RSGRAD_BSLICE_NW=8 python scripts/bench_paper.py bslice
python scripts/bench_layer.py 64 10 bslice_bwd
