"""bslice fwd+bwd at a given grid (default the paper's 32x32x8 at 4 x 1024^2), for ncu / timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1904_12228_b200 import rsgrad as rs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
G = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
b = synth.bslice_inputs(N, 1024, 1024, 8, G, G, cfg=4, device="cuda")
out = (torch.empty_like(b["grid"]), torch.empty_like(b["guide"]), torch.empty_like(b["x"]))
fn = lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], out=out)
fn(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fn()
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / reps
print(f"bslice_bwd N={N} grid {G}x{G}x8: {t*1e3:.1f} us  ({N*1024*1024/t/1e3:.0f} Mpix/s, roofline {44*N*1024*1024/(t*1e-3)/1e9/6544:.3f})")
