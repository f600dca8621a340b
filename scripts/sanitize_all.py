"""Every C-ABI entry point and algorithm variant once on small / ragged shapes, for
compute-sanitizer (memcheck / racecheck): python scripts/sanitize_all.py."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1904_12228_b200 import rsgrad as rs

dev = torch.device("cuda")
c = lambda d: {k: v.to(dev) for k, v in d.items()}  # noqa: E731
for shape in [(2, 5, 37, 53, 41, 29), (1, 16, 96, 128, 96, 128), (2, 4, 512, 512, 512, 512)]:
    N, C, H, W, Ho, Wo = shape
    s = c(synth.stn_inputs(N, C, H, W, Ho, Wo, cfg=1))
    for pad in ("zeros", "border"):
        rs.stn_fwd(s["x"], s["theta"], Ho, Wo, padding=pad)
        for algo in (("auto", "scatter_priv", "scatter_atomic") if pad == "border" else
                     ("auto", "gather", "scatter_priv", "scatter_atomic")):
            rs.stn_bwd(s["x"], s["theta"], s["dy"], padding=pad, algo=algo)
        rs.stn_bwd(s["x"], s["theta"], s["dy"], padding=pad, deterministic=True)
    th = s["theta"].clone()
    th[0] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])  # singular: fallback sample
    rs.stn_bwd(s["x"], th, s["dy"])
    rs.stn_bwd(s["x"], th, s["dy"], deterministic=True)
    rs.stn_bicubic_fwd(s["x"], s["theta"], Ho, Wo)
    rs.stn_bicubic_bwd(s["x"], th, s["dy"], deterministic=True)
    rs.stn_lanczos_bwd(s["x"], s["theta"], s["dy"])
    rs.stn_lanczos_bwd(s["x"], s["theta"], s["dy"], deterministic=True)
    rs.stn_lanczos_fwd(s["x"], s["theta"], Ho, Wo)
    for algo in ("auto", "gather"):
        rs.stn_bicubic_bwd(s["x"], s["theta"], s["dy"], algo=algo)
for flow in ("smooth", "stress"):
    w = c(synth.warp_inputs(2, 3, 45, 70, cfg=1, flow=flow))
    for pad in ("zeros", "border"):
        rs.warp_fwd(w["x"], w["flow"], padding=pad)
        for algo in ("auto", "scatter_priv", "scatter_atomic"):
            rs.warp_bwd(w["x"], w["flow"], w["dy"], padding=pad, algo=algo)
        rs.warp_bwd(w["x"], w["flow"], w["dy"], padding=pad, deterministic=True)
    for var in ("win8,4,4", "direct"):
        os.environ["RSGRAD_WARP_BWD"] = var
        rs.warp_bwd(w["x"], w["flow"], w["dy"])
        del os.environ["RSGRAD_WARP_BWD"]
    os.environ["RSGRAD_WARP_R"] = "8"
    rs.warp_bwd(w["x"], w["flow"], w["dy"])
    del os.environ["RSGRAD_WARP_R"]
for dims in [(2, 100, 130, 8, 6, 7), (1, 300, 260, 5, 3, 2), (1, 16, 16, 8, 16, 16)]:
    b = c(synth.bslice_inputs(*dims, cfg=1, grid="iid", guide="wide"))
    rs.bslice_fwd(b["grid"], b["guide"], b["x"])
    for algo in ("auto", "scatter_atomic"):
        rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], algo=algo)
    rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], deterministic=True)
x = torch.randn(2, 9, 37, 45, device=dev)
k = torch.randn(17, 9, 3, 5, device=dev)
dy = torch.randn(2, 17, 37, 45, device=dev)
rs.conv_fwd(x, k)
for algo in ("auto", "scatter_atomic"):
    rs.conv_bwd(x, k, dy, algo=algo)
inp, tgt = torch.randn(2, 45, 70, device=dev), torch.randn(2, 45, 70, device=dev)
for sch in ("root", "inline", "at"):
    rs.convloss_grad(inp, torch.randn(3, 5), tgt, schedule=sch)
u = torch.randn(1, 3, 5, 7, device=dev)
rs.upsample4_bwd(rs.upsample4_fwd(u))
x3 = torch.randn(1, 2, 9, 11, 13, device=dev)
t3 = torch.eye(3, 4, device=dev)[None] + 0.05 * torch.randn(1, 3, 4, device=dev)
rs.stn3d_bwd(x3, t3, rs.stn3d_fwd(x3, t3))
rs.stn3d_bwd(x3, t3, rs.stn3d_fwd(x3, t3), deterministic=True)
torch.cuda.synchronize()
print("sanitize_all: done")
