"""e2e (host-buffer) step timing under several host-pipeline settings, one process."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1904_12228_b200 import rsgrad as rs

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
settings = [s.split(":") for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8:2", "16:3"])]
s, w, b = bench.make_inputs(0, nb, torch.device("cuda"))
pick = lambda d: {k: v.cpu().pin_memory() for k, v in d.items()}  # noqa: E731
hs, hw, hb = pick(s), pick(w), pick(b)
del s, w, b
torch.cuda.empty_cache()
ho = bench.alloc_outputs(hs, hw, hb, host=True)
calls = bench.step_calls(rs, hs, hw, hb, ho, sync=False)
for ch, ns in settings:
    os.environ["RSGRAD_HOST_CHUNKS"], os.environ["RSGRAD_HOST_STREAMS"] = ch, ns
    for _, fn in calls:
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        for _, fn in calls:
            fn()
        torch.cuda.current_stream().synchronize()
    dt = (time.perf_counter() - t0) / 2
    per = {}
    for name, fn in calls:
        t1 = time.perf_counter(); fn(); torch.cuda.current_stream().synchronize(); per[name] = time.perf_counter() - t1
    print(f"chunks {ch:>3s} streams {ns}: step {dt*1e3:.0f} ms -> {nb*1024*1024/dt/1e6:.1f} Mpix/s  "
          + " ".join(f"{k}={v*1e3:.0f}" for k, v in per.items()), flush=True)
