"""Row a11 evidence: every d_input / d_grid algorithm of each layer once per repetition on
the configs[4] shapes at NB samples (default 8), timed with CUDA events (median of REPS);
under ncu (`--set full --metrics <atomic counters>`) the same script yields the counters
per variant.  python scripts/prof_a11.py [NB] [REPS] > out.json"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1904_12228_b200 import rsgrad as rs

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1  # run one variant (per-variant ncu reports)
dev = torch.device("cuda")
s, w, b = bench.make_inputs(0, nb, dev)
o = bench.alloc_outputs(s, w, b)


def env(k, v):
    def f():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    return f


variants = [
    ("stn_bwd", "AUTO (cell-owner gather + d_theta tiles)", None,
     lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"], out=(o["stn_dx"], o["stn_dth"]))),
    ("stn_bwd", "SCATTER_PRIV (shared float atomics + flush reds)", None,
     lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"], algo="scatter_priv", out=(o["stn_dx"], o["stn_dth"]))),
    ("stn_bwd", "SCATTER_ATOMIC (per-tap global reds)", None,
     lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"], algo="scatter_atomic", out=(o["stn_dx"], o["stn_dth"]))),
    ("warp_bwd", "AUTO (row strips, register-combined reds)", None,
     lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], out=(o["warp_dx"], o["warp_df"]))),
    ("warp_bwd", "SCATTER_ATOMIC (one red per tap)", None,
     lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], algo="scatter_atomic", out=(o["warp_dx"], o["warp_df"]))),
    ("warp_bwd", "SCATTER_PRIV (shared footprint + flush reds)", None,
     lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], algo="scatter_priv", out=(o["warp_dx"], o["warp_df"]))),
    ("warp_bwd", "windows (per-warp smem windows, red.v4 flush)", ("RSGRAD_WARP_BWD", "win8,4,4"),
     lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], out=(o["warp_dx"], o["warp_df"]))),
    ("warp_bwd", "deterministic (fixed-point int64 scatter)", None,
     lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], deterministic=True, out=(o["warp_dx"], o["warp_df"]))),
    ("bslice_bwd", "AUTO (dual-cell register accumulation + partial gather)", None,
     lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], out=(o["bs_dgr"], o["bs_dgd"], o["bs_dx"]))),
    ("bslice_bwd", "GATHER (pure node gather: each node walks its 2x2 dual cells)", None,
     lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], algo="gather",
                           out=(o["bs_dgr"], o["bs_dgd"], o["bs_dx"]))),
    ("bslice_bwd", "SCATTER_ATOMIC (per-pixel global reds into d_grid)", None,
     lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], algo="scatter_atomic",
                           out=(o["bs_dgr"], o["bs_dgd"], o["bs_dx"]))),
]
res = []
for vi, (call, name, ev, fn) in enumerate(variants):
    if only >= 0 and vi != only:
        continue
    if ev:
        os.environ[ev[0]] = ev[1]
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    if ev:
        os.environ.pop(ev[0], None)
    res.append({"call": call, "variant": name, "ms": round(statistics.median(ts), 4), "samples": nb})
    print(json.dumps(res[-1]), flush=True)
