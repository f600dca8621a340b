# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err; tail -c 300 gpurun_out/bench_r2k.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_r2k.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/paper_r2k.csv python scripts/bench_paper.py --launches gpurun_out/paper_r2k.csv.order > gpurun_out/pl.log 2>&1
python scripts/bench_paper.py --parse gpurun_out/paper_r2k.csv > gpurun_out/paper_breakdown_r2k.md 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
