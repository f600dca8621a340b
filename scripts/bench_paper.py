"""bench.py's paper_shapes() alone (configs[1..3] + the paper's bslice grids, L2 flushed
per call): python scripts/bench_paper.py [filter]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1904_12228_b200 import rsgrad as rs

res = bench.paper_shapes(rs, bench.peak_hbm()[0])
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in res["cases"].items():
    if flt in k:
        print(f"{k:32s} fwd {v['fwd_us']:8.1f} us ({v['fwd_roofline_frac']:.3f})  bwd {v['bwd_us']:8.1f} us ({v['bwd_roofline_frac']:.3f})")
