"""Timing of the §8(f) rows at the paper's shapes (CUDA events, L2 flushed before each call)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_12228_b200 import rsgrad as rs

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def conv_case(N=16, C=16, H=256, W=256, k=3):
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(N, C, H, W, device=dev, generator=g)
    kk = torch.randn(C, C, k, k, device=dev, generator=g) / (C * k * k) ** 0.5
    dy = torch.randn(N, C, H, W, device=dev, generator=g)
    y = torch.empty_like(x); dx = torch.empty_like(x); dk = torch.empty_like(kk)
    r = {"fwd_ms": timed(lambda: rs.conv_fwd(x, kk, out=y)),
         "bwd_gather_ms": timed(lambda: rs.conv_bwd(x, kk, dy, out=(dx, dk))),
         "bwd_dx_gather_ms": timed(lambda: rs.conv_bwd(x, kk, dy, need_dk=False, out=(dx, None))),
         "bwd_dk_ms": timed(lambda: rs.conv_bwd(x, kk, dy, need_dx=False, out=(None, dk))),
         "bwd_dx_atomic_ms": timed(lambda: rs.conv_bwd(x, kk, dy, algo="scatter_atomic", need_dk=False,
                                                        out=(dx, None)), reps=5)}
    fl = 2.0 * N * H * W * C * C * k * k
    r["fwd_tflops"] = fl / r["fwd_ms"] / 1e9
    r["dx_gather_tflops"] = fl / r["bwd_dx_gather_ms"] / 1e9
    r["dk_tflops"] = fl / r["bwd_dk_ms"] / 1e9
    return r


if __name__ == "__main__":
    print(json.dumps({"conv_16x16x256x256_k3": conv_case()}, indent=1))
