# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -k "lanczos" > gpurun_out/pytest_lz.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_lz.log
python -c "
import bench, json
from paper_1904_12228_b200 import rsgrad as rs
r = bench.next_rows(rs, bench.peak_hbm()[0])['rows']
print(json.dumps({k: v for k, v in r.items() if 'lanczos' in k}))"
