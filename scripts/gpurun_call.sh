timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/b_ncu.log 2>&1; echo ncu=$?
PROF_CMD="python scripts/bench_next.py" bash scripts/gpurun_prof.sh convp "conv_direct|conv_dk_partial|conv_dx_atomic" 2 RS_X=1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/bench.json
