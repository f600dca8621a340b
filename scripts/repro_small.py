import sys; sys.path.insert(0,'.')
import torch, synth
from paper_1904_12228_b200 import rsgrad
inp = synth.stn_inputs(2, 3, 32, 48, cfg=1, theta_kind="identity")
g = {k: v.cuda().contiguous() for k, v in inp.items()}
dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
torch.cuda.synchronize(); print("ok", float(dx.abs().sum()))
