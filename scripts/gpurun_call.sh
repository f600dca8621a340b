# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pt_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pt_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-paper-shapes --no-cpu --no-e2e --no-next > gpurun_out/r2_launch_bench.log 2>&1
python scripts/launch_shares.py gpurun_out/r2_launches.csv > gpurun_out/r2_launch_shares.md 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_final.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])
for k,v in d['layers'].items(): print(k, v)
for k,v in d['paper_shapes']['cases'].items(): print(k, v['fwd_us'], v['bwd_us'], v['fwd_roofline_frac'], v['bwd_roofline_frac'])
"
