"""Run each C-ABI call once at a given scale with a sync after each (debug aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1904_12228_b200 import rsgrad as rs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda")
def run(name, fn):
    t = time.time()
    fn(); torch.cuda.synchronize()
    print(f"{name:12s} ok {time.time()-t:.3f}s", flush=True)
s = synth.stn_inputs(N, 16, S, S, cfg=5, device=dev)
run("stn_fwd", lambda: rs.stn_fwd(s["x"], s["theta"]))
run("stn_bwd", lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"]))
del s
w = synth.warp_inputs(N, 3, S, S, cfg=5, device=dev)
run("warp_fwd", lambda: rs.warp_fwd(w["x"], w["flow"]))
run("warp_bwd", lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"]))
b = synth.bslice_inputs(N, S, S, 8, 16, 16, cfg=5, device=dev)
run("bslice_fwd", lambda: rs.bslice_fwd(b["grid"], b["guide"], b["x"]))
run("bslice_bwd", lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"]))
