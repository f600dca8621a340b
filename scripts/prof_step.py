"""One bench step (all six calls) at a reduced batch, for ncu: warm-up step then one profiled step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1904_12228_b200 import rsgrad as rs

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda")
s, w, b = bench.make_inputs(0, nb, dev)
o = bench.alloc_outputs(s, w, b)
calls = bench.step_calls(rs, s, w, b, o)
for _ in range(reps):
    for _, fn in calls:
        fn()
torch.cuda.synchronize()
print("done", nb)
