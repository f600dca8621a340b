import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1904_12228_b200 import rsgrad as rs
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256
s = synth.stn_inputs(N, 16, S, S, cfg=5, device="cuda")
rs.launch_count(reset=True)
dx, dth = rs.stn_bwd(s["x"], s["theta"], s["dy"])
torch.cuda.synchronize()
print("launches", rs.launch_count(), "err", rs.lib().rsgrad_last_error())
ws = rs.workspace_bytes(0, N, 16, S, S, S, S)
print("ws bytes", ws)
