import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1904_12228_b200 import rsgrad as rs
N, S, G = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
b = synth.bslice_inputs(N, S, S, 8, G, G, cfg=5, device="cuda")
rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"]); torch.cuda.synchronize(); print("ok", N, S, G)
