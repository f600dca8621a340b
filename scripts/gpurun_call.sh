mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn or graph or warp_determ" > gpurun_out/pytest_stn$i.log 2>&1; tail -1 gpurun_out/pytest_stn$i.log; done
grep -E "^FAILED" gpurun_out/pytest_stn*.log | head
python scripts/bench_layer.py 64 10 stn_bwd; python scripts/bench_paper.py stn
timeout 600 python bench.py --no-paper-shapes --no-next --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
