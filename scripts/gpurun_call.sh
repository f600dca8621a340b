timeout 900 python -m pytest tests -m gpu -q -x -k "stn3d or bench_shapes_sampled" > gpurun_out/pytest_3d.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_3d.log
python -c "
import bench, json
from paper_1904_12228_b200 import rsgrad as rs
r = bench.next_rows(rs, bench.peak_hbm()[0])['rows']
print(json.dumps({k: v for k, v in r.items() if k.startswith('f3')}, indent=1))"
