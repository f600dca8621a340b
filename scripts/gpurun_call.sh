timeout 900 python -m pytest tests -m gpu -q -k "conv or upsample or bicubic or stn3d or variants" > gpurun_out/pytest_f.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_f.log
python -c "
import bench, json
from paper_1904_12228_b200 import rsgrad as rs
print(json.dumps(bench.next_rows(rs, bench.peak_hbm()[0]), indent=1))" > gpurun_out/next.json 2>&1; cat gpurun_out/next.json
