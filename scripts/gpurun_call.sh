mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or graph" > gpurun_out/pytest_stn.log 2>&1; tail -2 gpurun_out/pytest_stn.log
for f in 4096 0; do echo fork=$f; RSGRAD_STN_FORK=$f python scripts/bench_paper.py stn; done
python scripts/bench_layer.py 64 10 stn_bwd
for nb in 4 8 16; do for f in 100000 0; do echo nb=$nb fork=$f; RSGRAD_STN_FORK=$f python scripts/bench_layer.py $nb 20 stn_bwd; done; done
