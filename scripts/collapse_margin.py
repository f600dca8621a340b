"""Margin of the AUTO warp d_input against T on the collapsing flow at configs[2]'s shape
(the atomic order varies run to run): max_ratio over REPS runs, both paddings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, synth, oracle
from paper_1904_12228_b200 import rsgrad as rs
from _tol import compare, GRAD
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
N, C, H, W = 8, 3, 384, 512
inp = synth.warp_inputs(N, C, H, W, cfg=3, flow="smooth")
yy, xx = torch.meshgrid(torch.arange(H, dtype=torch.float32), torch.arange(W, dtype=torch.float32), indexing="ij")
inp["flow"] = torch.stack([-xx * 0.97 + 3.3, -yy * 0.9 + 2.6]).expand(N, 2, H, W).contiguous()
g = {k: v.cuda() for k, v in inp.items()}
for pad in ("zeros", "border"):
    rdx, _ = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")), pad == "border")
    for algo in ("auto", "scatter_atomic", "deterministic"):
        kw = {"deterministic": True} if algo == "deterministic" else {"algo": algo}
        rat = [compare(rs.warp_bwd(g["x"], g["flow"], g["dy"], padding=pad, **kw)[0].double().cpu().numpy(), rdx,
                       **GRAD)["max_ratio"] for _ in range(reps)]
        print(f"{pad:6s} {algo:15s} max_ratio over {reps} runs: max {max(rat):.3f} min {min(rat):.3f}")
