"""bench.py's paper_shapes() alone (configs[1..3] + the paper's bslice grids, L2 flushed
per call, eager and CUDA-graph): python scripts/bench_paper.py [filter]

  --launches   no timing: flush, fwd, flush, bwd per case (twice), for an ncu launch list
               (ncu --metrics gpu__time_duration.sum --csv --log-file F python ... --launches)
  --parse F    per-kernel breakdown of that launch list, one table per call (markdown)"""
import collections, csv, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if "--parse" in sys.argv:
    f = sys.argv[sys.argv.index("--parse") + 1]
    rows = list(csv.reader([l for l in open(f) if l.startswith('"')]))
    h = rows[0]; iN = h.index("Kernel Name"); iV = h.index("Metric Value"); iU = h.index("Metric Unit")
    seq = []
    for r in rows[1:]:
        k = r[iN].split('(')[0].replace('<unnamed>::', '').replace('void ', '').replace('rs::', '')
        v = float(r[iV]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iU], 1.0)
        seq.append((k, v))
    # segments: every non-library kernel is the L2 flush that opens a call
    calls, cur = [], None
    for k, v in seq:
        if "elementwise" in k or "at::" in k:
            cur = []
            calls.append(cur)
        elif cur is not None:
            cur.append((k, v))
    calls = [c for c in calls if c]
    names = open(f + ".order").read().split() if os.path.exists(f + ".order") else [str(i) for i in range(len(calls))]
    agg = collections.OrderedDict()
    for nm, c in zip(names, calls):
        agg.setdefault(nm, []).append(c)
    for nm, reps in agg.items():
        last = reps[-1]
        print(f"\n**{nm}** ({len(last)} launches, kernel sum {sum(v for _, v in last):.1f} us)\n")
        print("| kernel | us |\n|---|---|")
        for k, v in last:
            print(f"| {k} | {v:.1f} |")
    sys.exit(0)

import torch
import bench
from paper_1904_12228_b200 import rsgrad as rs

if "--launches" in sys.argv:
    dev = torch.device("cuda")
    fl = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    order = []
    for name, layer, C, P, fwd, bwd in bench.paper_cases(rs, dev):
        for rep in range(2):
            for kind, fn in (("fwd", fwd), ("bwd", bwd)):
                bench.flush_l2(fl)
                fn()
                order.append(f"{name}.{kind}")
    torch.cuda.synchronize()
    out = sys.argv[sys.argv.index("--launches") + 1] if len(sys.argv) > sys.argv.index("--launches") + 1 else None
    if out:
        open(out, "w").write("\n".join(order))
    sys.exit(0)

res = bench.paper_shapes(rs, bench.peak_hbm()[0])
flt = next((a for a in sys.argv[1:] if not a.startswith("-")), "")
for k, v in res["cases"].items():
    if flt in k:
        print(f"{k:30s} fwd {v['fwd_us']:7.1f} graph {v['fwd_us_graph']:7.1f} us  "
              f"bwd {v['bwd_us']:7.1f} graph {v['bwd_us_graph']:7.1f} us  "
              f"(fracs {v['fwd_roofline_frac']:.3f} / {v['bwd_roofline_frac']:.3f})")
