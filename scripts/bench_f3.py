"""bench.py's next_rows() alone (the SURVEY 8(f) rows, L2 flushed per call): python scripts/bench_f3.py [filter]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1904_12228_b200 import rsgrad as rs

res = bench.next_rows(rs, bench.peak_hbm()[0])
flt = next((a for a in sys.argv[1:] if not a.startswith("-")), "")
for k, v in res["rows"].items():
    if flt in k:
        print(k, json.dumps({a: b for a, b in v.items() if "us" in a}))
