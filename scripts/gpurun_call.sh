mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bslice" > gpurun_out/pytest_bs.log 2>&1; tail -1 gpurun_out/pytest_bs.log
python scripts/bench_layer.py 64 10 bslice_fwd; python scripts/bench_paper.py bslice
