import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth, oracle
from paper_1904_12228_b200 import rsgrad as rs
N, C, H, W = 8, 3, 384, 512
inp = synth.warp_inputs(N, C, H, W, cfg=3, flow="smooth")
yy, xx = torch.meshgrid(torch.arange(H, dtype=torch.float32), torch.arange(W, dtype=torch.float32), indexing="ij")
inp["flow"] = torch.stack([-xx * 0.97 + 3.3, -yy * 0.9 + 2.6]).expand(N, 2, H, W).contiguous()
g = {k: v.cuda() for k, v in inp.items()}
x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
rdx, _ = oracle.warp_bwd(x, fl, dy, True)
absdx, _ = oracle.warp_bwd(x, fl, np.abs(dy), True)
s = max(1.0, float(np.sqrt(np.mean(rdx * rdx))))
for R in ("8", "16"):
    os.environ["RSGRAD_WARP_R"] = R
    dx = rs.warp_bwd(g["x"], g["flow"], g["dy"], padding="border")[0].double().cpu().numpy()
    dd = rs.warp_bwd(g["x"], g["flow"], g["dy"], padding="border", deterministic=True)[0].double().cpu().numpy()
    err = np.abs(dx - rdx); bound = 1e-4 * np.abs(rdx) + 1e-6 * s
    i = np.unravel_index(np.argmax(err / bound), err.shape)
    print("R", R, "rms", s, "worst", i, "r", rdx[i], "gpu", dx[i], "det", dd[i], "err", err[i], "ratio", (err / bound)[i],
          "sum|terms|", absdx[i], "deterr", abs(dd[i] - rdx[i]))
    top = np.argsort((err / bound).ravel())[-5:]
    print("  top ratios", (err / bound).ravel()[top], "abs r", np.abs(rdx.ravel()[top]), "sum|t|", absdx.ravel()[top])
