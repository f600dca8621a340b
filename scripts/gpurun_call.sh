# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "host or workspace or deterministic" > gpurun_out/r2_pt_host.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pt_host.log
timeout 900 python bench.py --no-next --no-paper-shapes --no-cpu > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'])"
bash scripts/sanitize_run.sh
