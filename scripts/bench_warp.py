"""warp_bwd at the paper shape (8x3x384x512, smooth / stress) and configs[4] shapes, per variant env.
python scripts/bench_warp.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1904_12228_b200 import rsgrad as rs
dev = torch.device("cuda")
fl = torch.zeros(64 * 1024 * 1024, device=dev)
for name, N, H, W in (("K3", 8, 384, 512), ("K5/4", 16, 1024, 1024)):
    for flow in ("smooth", "stress"):
        i = synth.warp_inputs(N, 3, H, W, cfg=3, device=dev, flow=flow)
        o = (torch.empty_like(i["x"]), torch.empty_like(i["flow"]))
        ts = []
        for r in range(15):
            fl.add_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); rs.warp_bwd(i["x"], i["flow"], i["dy"], out=o); e1.record(); torch.cuda.synchronize()
            if r >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{name} {flow:7s} {statistics.median(ts):8.1f} us")
