timeout 900 python -m pytest tests -m gpu -q -x -k "stn" > gpurun_out/pytest_stn.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_stn.log
for i in 1 2; do
echo "== concurrent"; python scripts/bench_layer.py 16 5 stn_bwd
echo "== serial"; RSGRAD_STN_CONCURRENT=0 python scripts/bench_layer.py 16 5 stn_bwd
done
echo "== concurrent 64"; python scripts/bench_layer.py 64 3 stn_bwd
echo "== serial 64"; RSGRAD_STN_CONCURRENT=0 python scripts/bench_layer.py 64 3 stn_bwd
