"""Pinned H2D / D2H bandwidth alone and concurrently (two streams)."""
import torch, time
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d(): d.copy_(h, non_blocking=True)
def d2h(): h.copy_(d, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
gb = n * 4 / 1e9
print(f"H2D {gb / t(h2d):.1f} GB/s, D2H {gb / t(d2h):.1f} GB/s, concurrent {2 * gb / t(both):.1f} GB/s total")
