"""Which host call breaks a global-mode stream capture of the C-ABI calls?"""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from cuda.bindings import runtime as cr
from paper_1904_12228_b200 import rsgrad as rs

x = torch.randn(1 << 20, device="cuda")


def probe(name, fn, mode="global"):
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, capture_error_mode=mode):
            fn()
        print(f"{name:40s} {mode:8s} OK", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name:40s} {mode:8s} FAIL {str(e).splitlines()[0][:100]}", flush=True)
    torch.cuda.synchronize()


probe("torch add", lambda: x.add_(1))
probe("cudaPointerGetAttributes", lambda: cr.cudaPointerGetAttributes(x.data_ptr()))
probe("cudaGetDevice", lambda: cr.cudaGetDevice())
probe("cudaStreamGetDevice", lambda: cr.cudaStreamGetDevice(torch.cuda.current_stream().cuda_stream))
probe("cudaDeviceGetAttribute", lambda: cr.cudaDeviceGetAttribute(cr.cudaDeviceAttr.cudaDevAttrMultiProcessorCount, 0))
probe("cudaGetLastError", lambda: cr.cudaGetLastError())
th = torch.zeros(4, 2, 3, device="cuda"); th[:, 0, 0] = 1; th[:, 1, 1] = 1
xi = torch.randn(4, 16, 512, 512, device="cuda"); y = torch.empty_like(xi)
rs.stn_fwd(xi, th, out=y); torch.cuda.synchronize()
for mode in ("global", "thread_local", "relaxed"):
    probe("rs.stn_fwd", lambda: rs.stn_fwd(xi, th, out=y), mode)
