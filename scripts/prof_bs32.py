"""bslice_bwd at the paper's 1024^2 / 32x32x8 shape (K4'), for ncu: warm-up + one call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1904_12228_b200 import rsgrad as rs
i = synth.bslice_inputs(4, 1024, 1024, 8, 32, 32, cfg=4, device=torch.device("cuda"))
for _ in range(2):
    rs.bslice_bwd(i["grid"], i["guide"], i["x"], i["dy"])
torch.cuda.synchronize()
