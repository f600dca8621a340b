"""Quick per-call timing at the configs[4] shapes (batch nb): events, warm L2 irrelevant (>L2)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1904_12228_b200 import rsgrad as rs

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
only = sys.argv[3].split(",") if len(sys.argv) > 3 else None
dev = torch.device("cuda")
s, w, b = bench.make_inputs(0, nb, dev)
o = bench.alloc_outputs(s, w, b)
calls = bench.step_calls(rs, s, w, b, o)
peak = bench.peak_hbm()[0]
P = nb * bench.H * bench.W
res = {}
for name, fn in calls:
    if only and not any(k in name for k in only):
        continue
    fn(); fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    res[name] = {"ms": round(t * 1e3, 3), "frac": round(bench.CALL_BYTES[name] * P / t / 1e9 / peak, 3)}
    print(f"{name:12s} {t*1e3:8.3f} ms  roofline {res[name]['frac']:.3f}", flush=True)

if os.environ.get("RS_BENCH_ALGOS"):
    # d_input algorithm comparison per layer (AUTO vs SCATTER_PRIV vs SCATTER_ATOMIC)
    for algo in ("auto", "scatter_priv", "scatter_atomic"):
        for name, fn in [("stn_bwd", lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"], algo=algo, out=(o["stn_dx"], o["stn_dth"]))),
                         ("warp_bwd", lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], algo=algo, out=(o["warp_dx"], o["warp_df"])))]:
            fn(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record(); torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / reps * 1e-3
            print(f"{name:10s} {algo:15s} {t*1e3:8.3f} ms  roofline {bench.CALL_BYTES[name] * P / t / 1e9 / peak:.3f}", flush=True)
