mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or graph" > gpurun_out/pytest_stn$i.log 2>&1; tail -1 gpurun_out/pytest_stn$i.log; done
grep -E "^FAILED" gpurun_out/pytest_stn1.log | head
python scripts/bench_layer.py 64 10 stn_bwd; python scripts/bench_paper.py stn
