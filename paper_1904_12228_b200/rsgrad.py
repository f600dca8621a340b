"""Thin Python binding of the rsgrad C ABI (include/rsgrad.h).

Argument marshalling only: every step of every layer runs in the CUDA kernels
of ``librsgrad.so``.  There is no CPU or PyTorch fallback: if the library is
missing (and cannot be built) or no CUDA device is present, calls raise.

Functions take float32 C-contiguous torch tensors.  CUDA tensors are passed as
device pointers on the current torch stream; CPU tensors (pinned or pageable)
are passed as host pointers and the library stages them;
for CPU outputs the call synchronises the stream before returning.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _build

_PADDING = {"zeros": 0, "border": 1}
_ALGO = {"auto": 0, "gather": 1, "scatter_priv": 2, "scatter_atomic": 3}
LAYER_STN, LAYER_WARP, LAYER_BSLICE, LAYER_CONV = 0, 1, 2, 3
LAYER_BICUBIC, LAYER_STN3D, LAYER_LANCZOS = 5, 6, 7  # rsgrad_bwd_workspace_bytes layer ids


class RsOpts(ctypes.Structure):
    _fields_ = [("align_corners", ctypes.c_int), ("padding", ctypes.c_int),
                ("algo", ctypes.c_int), ("deterministic", ctypes.c_int)]


class RsgradError(RuntimeError):
    pass


_lib = None


def lib():
    """Load librsgrad.so (building it in-tree if stale and nvcc is available)."""
    global _lib
    if _lib is None:
        path = _build.LIB
        try:
            # RSGRAD_LIB: an alternative build of the same library (A/B timing, sanitizer
            # builds); default: the in-tree librsgrad.so, rebuilt if stale
            path = os.environ.get("RSGRAD_LIB") or _build.build()
        except (OSError, FileNotFoundError, Exception) as e:  # noqa: BLE001
            if not os.path.exists(_build.LIB):
                raise RsgradError(f"librsgrad.so is missing and could not be built: {e}") from e
        L = ctypes.CDLL(path)
        P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        O = ctypes.POINTER(RsOpts)
        L.stn_fwd.argtypes = [P, P, I, I, I, I, I, I, O, P, P]
        L.stn_bwd.argtypes = [P, P, P, I, I, I, I, I, I, O, P, P, P, S, P]
        L.warp_fwd.argtypes = [P, P, I, I, I, I, O, P, P]
        L.warp_bwd.argtypes = [P, P, P, I, I, I, I, O, P, P, P, S, P]
        L.bslice_fwd.argtypes = [P, P, P, I, I, I, I, I, I, O, P, P]
        L.bslice_bwd.argtypes = [P, P, P, P, I, I, I, I, I, I, O, P, P, P, P, S, P]
        L.conv_fwd.argtypes = [P, P, I, I, I, I, I, I, I, O, P, P]
        L.convloss_grad.argtypes = [P, P, P, I, I, I, I, I, I, P, P, S, P]
        L.upsample4_fwd.argtypes = [P, I, I, I, I, P, P]
        L.stn_bicubic_fwd.argtypes = [P, P, I, I, I, I, I, I, O, P, P]
        L.stn_bicubic_bwd.argtypes = [P, P, P, I, I, I, I, I, I, O, P, P, P, S, P]
        L.stn_lanczos_fwd.argtypes = [P, P, I, I, I, I, I, I, O, P, P]
        L.stn_lanczos_bwd.argtypes = [P, P, P, I, I, I, I, I, I, O, P, P, P, S, P]
        L.stn3d_fwd.argtypes = [P, P, I, I, I, I, I, I, I, I, O, P, P]
        L.stn3d_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, I, O, P, P, P, S, P]
        L.upsample4_bwd.argtypes = [P, I, I, I, I, P, P]
        L.conv_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, O, P, P, P, S, P]
        for f in ("stn_fwd", "stn_bwd", "warp_fwd", "warp_bwd", "bslice_fwd", "bslice_bwd", "conv_fwd", "conv_bwd",
                  "convloss_grad", "upsample4_fwd", "upsample4_bwd", "stn_bicubic_fwd", "stn_bicubic_bwd",
                  "stn3d_fwd", "stn3d_bwd", "stn_lanczos_fwd", "stn_lanczos_bwd"):
            getattr(L, f).restype = ctypes.c_int
        L.rsgrad_bwd_workspace_bytes.argtypes = [I, I, I, I, I, I, I, I, I, I, O]
        L.rsgrad_bwd_workspace_bytes.restype = S
        L.rsgrad_last_error.restype = ctypes.c_char_p
        L.rsgrad_version.restype = ctypes.c_char_p
        L.rsgrad_set_host_staging.argtypes = [P, S]
        L.rsgrad_set_host_staging.restype = ctypes.c_int
        L.rsgrad_launch_count.argtypes = [I]
        L.rsgrad_launch_count.restype = ctypes.c_ulonglong
        _lib = L
    return _lib


def version() -> str:
    return lib().rsgrad_version().decode()


def set_host_staging(buf):
    """Register a caller-owned CUDA uint8 tensor as the host-pointer path's staging
    buffer on this thread / its device (None: unregister).  Keep the tensor alive while
    registered."""
    if buf is None:
        _check(lib().rsgrad_set_host_staging(None, 0), "rsgrad_set_host_staging")
        return
    with torch.cuda.device(buf.device):
        _check(lib().rsgrad_set_host_staging(ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size()),
               "rsgrad_set_host_staging")


def launch_count(reset: bool = False) -> int:
    return int(lib().rsgrad_launch_count(int(reset)))


def _check(st: int, what: str):
    if st != 0:
        msg = lib().rsgrad_last_error().decode()
        raise RsgradError(f"{what} failed (status {st}): {msg}")


def _opts(align_corners=True, padding="zeros", algo="auto", deterministic=False):
    return RsOpts(int(bool(align_corners)), _PADDING[padding], _ALGO[algo], int(bool(deterministic)))


def _ptr(t):
    if t is None:
        return None
    if t.dtype != torch.float32:
        raise TypeError(f"expected float32 tensor, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _device_of(*ts):
    for t in ts:
        if t is not None and t.is_cuda:
            return t.device
    return None


def _stream(dev):
    if not torch.cuda.is_available():
        raise RsgradError("rsgrad needs a CUDA device (no CPU fallback)")
    s = torch.cuda.current_stream(dev) if dev is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _like(ref, shape):
    if ref.is_cuda:
        return torch.empty(shape, dtype=torch.float32, device=ref.device)
    return torch.empty(shape, dtype=torch.float32, pin_memory=torch.cuda.is_available())


def _sync_if_host(dev, sync, *outs):
    """Host outputs are written by async D2H copies on the stream: unless the caller
    passed sync=False (and synchronises the stream itself), wait for them."""
    if sync and any(o is not None and not o.is_cuda for o in outs):
        (torch.cuda.current_stream(dev) if dev is not None else torch.cuda.current_stream()).synchronize()


def _workspace(dev, nbytes):
    if nbytes == 0:
        return None, 0
    d = dev if dev is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.empty(nbytes, dtype=torch.uint8, device=d), nbytes


def _wsp(ws):
    return None if ws is None else ctypes.c_void_p(ws.data_ptr())


def workspace_bytes(layer, N, C=0, H=0, W=0, Ho=0, Wo=0, D=0, Gh=0, Gw=0, opts=None):
    o = opts if opts is not None else _opts()
    return int(lib().rsgrad_bwd_workspace_bytes(layer, N, C, H, W, Ho, Wo, D, Gh, Gw, ctypes.byref(o)))


# ----------------------------------------------------------------------------- STN
def stn_fwd(x, theta, Ho=None, Wo=None, *, align_corners=True, padding="zeros", out=None, sync=True):
    N, C, H, W = x.shape
    Ho = H if Ho is None else int(Ho)
    Wo = W if Wo is None else int(Wo)
    y = out if out is not None else _like(x, (N, C, Ho, Wo))
    dev = _device_of(x, theta, y)
    o = _opts(align_corners, padding)
    _check(lib().stn_fwd(_ptr(x), _ptr(theta), N, C, H, W, Ho, Wo, ctypes.byref(o), _ptr(y),
                         _stream(dev)), "stn_fwd")
    _sync_if_host(dev, sync, y)
    return y


def stn_bwd(x, theta, dy, *, align_corners=True, padding="zeros", algo="auto", deterministic=False,
            need_dx=True, need_dtheta=True, out=None, sync=True):
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    dx, dth = out if out is not None else (
        _like(x, (N, C, H, W)) if need_dx else None, _like(x, (N, 2, 3)) if need_dtheta else None)
    dev = _device_of(x, theta, dy, dx, dth)
    o = _opts(align_corners, padding, algo, deterministic)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_STN, N, C, H, W, Ho, Wo, opts=o))
    _check(lib().stn_bwd(_ptr(x), _ptr(theta), _ptr(dy), N, C, H, W, Ho, Wo, ctypes.byref(o),
                         _ptr(dx), _ptr(dth), None if ws is None else ctypes.c_void_p(ws.data_ptr()),
                         nws, _stream(dev)), "stn_bwd")
    _sync_if_host(dev, sync, dx, dth)
    return dx, dth


# ----------------------------------------------------------------------------- warp
def warp_fwd(x, flow, *, padding="zeros", out=None, sync=True):
    N, C, H, W = x.shape
    y = out if out is not None else _like(x, (N, C, H, W))
    dev = _device_of(x, flow, y)
    o = _opts(True, padding)
    _check(lib().warp_fwd(_ptr(x), _ptr(flow), N, C, H, W, ctypes.byref(o), _ptr(y), _stream(dev)),
           "warp_fwd")
    _sync_if_host(dev, sync, y)
    return y


def warp_bwd(x, flow, dy, *, padding="zeros", algo="auto", deterministic=False, need_dx=True,
             need_dflow=True, out=None, sync=True):
    N, C, H, W = x.shape
    dx, df = out if out is not None else (
        _like(x, (N, C, H, W)) if need_dx else None, _like(x, (N, 2, H, W)) if need_dflow else None)
    dev = _device_of(x, flow, dy, dx, df)
    o = _opts(True, padding, algo, deterministic)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_WARP, N, C, H, W, opts=o))
    _check(lib().warp_bwd(_ptr(x), _ptr(flow), _ptr(dy), N, C, H, W, ctypes.byref(o), _ptr(dx),
                          _ptr(df), None if ws is None else ctypes.c_void_p(ws.data_ptr()), nws,
                          _stream(dev)), "warp_bwd")
    _sync_if_host(dev, sync, dx, df)
    return dx, df


# ----------------------------------------------------------------------------- bslice
def bslice_fwd(grid, guide, x, *, out=None, sync=True):
    N, Q, D, Gh, Gw = grid.shape
    if Q != 12 or x.shape[1] != 3:
        raise ValueError("bslice: grid must be N x 12 x D x Gh x Gw and x N x 3 x H x W")
    H, W = guide.shape[1:]
    y = out if out is not None else _like(x, (N, 3, H, W))
    dev = _device_of(grid, guide, x, y)
    o = _opts()
    _check(lib().bslice_fwd(_ptr(grid), _ptr(guide), _ptr(x), N, H, W, D, Gh, Gw, ctypes.byref(o),
                            _ptr(y), _stream(dev)), "bslice_fwd")
    _sync_if_host(dev, sync, y)
    return y


def bslice_bwd(grid, guide, x, dy, *, algo="auto", deterministic=False, need_dgrid=True,
               need_dguide=True, need_dx=True, out=None, sync=True):
    N, Q, D, Gh, Gw = grid.shape
    H, W = guide.shape[1:]
    if out is not None:
        dgr, dgd, dx = out
    else:
        dgr = _like(x, (N, 12, D, Gh, Gw)) if need_dgrid else None
        dgd = _like(x, (N, H, W)) if need_dguide else None
        dx = _like(x, (N, 3, H, W)) if need_dx else None
    dev = _device_of(grid, guide, x, dy, dgr, dgd, dx)
    o = _opts(True, "zeros", algo, deterministic)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_BSLICE, N, 3, H, W, D=D, Gh=Gh, Gw=Gw, opts=o))
    _check(lib().bslice_bwd(_ptr(grid), _ptr(guide), _ptr(x), _ptr(dy), N, H, W, D, Gh, Gw,
                            ctypes.byref(o), _ptr(dgr), _ptr(dgd), _ptr(dx),
                            None if ws is None else ctypes.c_void_p(ws.data_ptr()), nws,
                            _stream(dev)), "bslice_bwd")
    _sync_if_host(dev, sync, dgr, dgd, dx)
    return dgr, dgd, dx


# ----------------------------------------------------------------------------- autograd
class SpatialTransformer(torch.autograd.Function):
    """y = grid_sample(x, affine_grid(theta)) with the rsgrad kernels."""

    @staticmethod
    def forward(ctx, x, theta, Ho=None, Wo=None, align_corners=True, padding="zeros"):
        x, theta = x.contiguous(), theta.contiguous()
        ctx.save_for_backward(x, theta)
        ctx.cfg = (align_corners, padding)
        return stn_fwd(x, theta, Ho, Wo, align_corners=align_corners, padding=padding)

    @staticmethod
    def backward(ctx, dy):
        x, theta = ctx.saved_tensors
        ac, pad = ctx.cfg
        dx, dth = stn_bwd(x, theta, dy.contiguous(), align_corners=ac, padding=pad,
                          need_dx=ctx.needs_input_grad[0], need_dtheta=ctx.needs_input_grad[1])
        return dx, dth, None, None, None, None


class FlowWarp(torch.autograd.Function):
    """FlowNet 2.0 warp y(x) = x_in(x + flow(x))."""

    @staticmethod
    def forward(ctx, x, flow, padding="zeros"):
        x, flow = x.contiguous(), flow.contiguous()
        ctx.save_for_backward(x, flow)
        ctx.padding = padding
        return warp_fwd(x, flow, padding=padding)

    @staticmethod
    def backward(ctx, dy):
        x, flow = ctx.saved_tensors
        dx, df = warp_bwd(x, flow, dy.contiguous(), padding=ctx.padding,
                          need_dx=ctx.needs_input_grad[0], need_dflow=ctx.needs_input_grad[1])
        return dx, df, None


class BilateralSlice(torch.autograd.Function):
    """HDRNet slice-apply."""

    @staticmethod
    def forward(ctx, grid, guide, x):
        grid, guide, x = grid.contiguous(), guide.contiguous(), x.contiguous()
        ctx.save_for_backward(grid, guide, x)
        return bslice_fwd(grid, guide, x)

    @staticmethod
    def backward(ctx, dy):
        grid, guide, x = ctx.saved_tensors
        n = ctx.needs_input_grad
        dgr, dgd, dx = bslice_bwd(grid, guide, x, dy.contiguous(), need_dgrid=n[0],
                                  need_dguide=n[1], need_dx=n[2])
        return dgr, dgd, dx


# ----------------------------------------------------------------------------- conv (§8(f) f1)
def conv_fwd(x, k, *, out=None):
    """y = 2-D convolution layer of PAPER.md:703-707 (include/rsgrad.h conv_fwd).
    CUDA tensors only (the kernel is shared by the batch)."""
    N, Ci, H, W = x.shape
    Co, Ci2, kh, kw = k.shape
    if Ci2 != Ci:
        raise ValueError("k must be Co x Ci x kh x kw")
    y = out if out is not None else _like(x, (N, Co, H, W))
    dev = _device_of(x, k, y)
    o = _opts()
    _check(lib().conv_fwd(_ptr(x), _ptr(k), N, Ci, Co, H, W, kh, kw, ctypes.byref(o), _ptr(y), _stream(dev)),
           "conv_fwd")
    return y


def conv_bwd(x, k, dy, *, algo="auto", deterministic=False, need_dx=True, need_dk=True, out=None):
    """(dx, dk): dx by the sheared gather (auto/gather) or the atomic scatter
    (scatter_atomic); dk by per-block partials + fixed-order sum."""
    N, Ci, H, W = x.shape
    Co, _, kh, kw = k.shape
    if out is not None:
        dx, dk = out
    else:
        dx = _like(x, (N, Ci, H, W)) if need_dx else None
        dk = _like(x, (Co, Ci, kh, kw)) if need_dk else None
    dev = _device_of(x, k, dy, dx, dk)
    o = _opts(True, "zeros", algo, deterministic)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_CONV, N, Ci, H, W, D=Co, Gh=kh, Gw=kw, opts=o))
    _check(lib().conv_bwd(_ptr(x), _ptr(k), _ptr(dy), N, Ci, Co, H, W, kh, kw, ctypes.byref(o), _ptr(dx), _ptr(dk),
                          None if ws is None else ctypes.c_void_p(ws.data_ptr()), nws, _stream(dev)), "conv_bwd")
    return dx, dk


# ----------------------------------------------------------------------------- §8(f) f4
_SCHED = {"root": 0, "inline": 1, "at": 2}
LAYER_CONVLOSS = 4


def convloss_grad(inp, k, target, *, schedule="root", out=None):
    """d_in of sum (conv(in, k) - target)^2; inp/target N x H x W CUDA
    tensors, k a kh x kw CPU tensor; schedule root / inline / at."""
    N, H, W = inp.shape
    kh, kw = k.shape
    kc = k.detach().to("cpu", torch.float32).contiguous()
    d = out if out is not None else torch.empty_like(inp)
    dev = _device_of(inp, target, d)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_CONVLOSS, N, 1, H, W) if schedule == "root" else 0)
    _check(lib().convloss_grad(_ptr(inp), _ptr(kc), _ptr(target), N, H, W, kh, kw, _SCHED[schedule], _ptr(d),
                               None if ws is None else ctypes.c_void_p(ws.data_ptr()), nws, _stream(dev)),
           "convloss_grad")
    return d


def upsample4_fwd(x, *, out=None):
    N, C, H, W = x.shape
    y = out if out is not None else torch.empty((N, C, 4 * H, 4 * W), dtype=torch.float32, device=x.device)
    _check(lib().upsample4_fwd(_ptr(x), N, C, H, W, _ptr(y), _stream(_device_of(x, y))), "upsample4_fwd")
    return y


def upsample4_bwd(dy, *, out=None):
    N, C, Ho, Wo = dy.shape
    if Ho % 4 or Wo % 4:
        raise ValueError("upsample4_bwd: d_output must be 4H x 4W")
    dx = out if out is not None else torch.empty((N, C, Ho // 4, Wo // 4), dtype=torch.float32, device=dy.device)
    _check(lib().upsample4_bwd(_ptr(dy), N, C, Ho // 4, Wo // 4, _ptr(dx), _stream(_device_of(dy, dx))),
           "upsample4_bwd")
    return dx


# ----------------------------------------------------------------------------- §8(f) f3
def stn_bicubic_fwd(x, theta, Ho=None, Wo=None, *, align_corners=True, out=None):
    """Bicubic STN (Keys A = -0.75, zeros); CUDA tensors."""
    N, C, H, W = x.shape
    Ho = H if Ho is None else int(Ho)
    Wo = W if Wo is None else int(Wo)
    y = out if out is not None else torch.empty((N, C, Ho, Wo), dtype=torch.float32, device=x.device)
    o = _opts(align_corners)
    _check(lib().stn_bicubic_fwd(_ptr(x), _ptr(theta), N, C, H, W, Ho, Wo, ctypes.byref(o), _ptr(y),
                                 _stream(_device_of(x, y))), "stn_bicubic_fwd")
    return y


def stn_bicubic_bwd(x, theta, dy, *, align_corners=True, algo="auto", deterministic=False, need_dx=True,
                    need_dtheta=True, out=None):
    """d_input by the converted gather over the affine preimage (gather, or deterministic=True)
    or the atomic scatter (auto / scatter_atomic); d_theta by fixed-order partial sums."""
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    if out is not None:
        dx, dth = out
    else:
        dx = torch.empty_like(x) if need_dx else None
        dth = torch.empty((N, 2, 3), dtype=torch.float32, device=x.device) if need_dtheta else None
    o = _opts(align_corners, "zeros", algo, deterministic)
    dev = _device_of(x, dy)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_BICUBIC, N, C, H, W, Ho, Wo, opts=o))
    _check(lib().stn_bicubic_bwd(_ptr(x), _ptr(theta), _ptr(dy), N, C, H, W, Ho, Wo, ctypes.byref(o), _ptr(dx),
                                 _ptr(dth), _wsp(ws), nws, _stream(dev)), "stn_bicubic_bwd")
    return dx, dth


def stn3d_fwd(x, theta, out_size=None, *, align_corners=True, out=None):
    """Volumetric STN (theta N x 3 x 4, trilinear, zeros); CUDA tensors."""
    N, C, D, H, W = x.shape
    Do, Ho, Wo = (D, H, W) if out_size is None else out_size
    y = out if out is not None else torch.empty((N, C, Do, Ho, Wo), dtype=torch.float32, device=x.device)
    o = _opts(align_corners)
    _check(lib().stn3d_fwd(_ptr(x), _ptr(theta), N, C, D, H, W, Do, Ho, Wo, ctypes.byref(o), _ptr(y),
                           _stream(_device_of(x, y))), "stn3d_fwd")
    return y


def stn3d_bwd(x, theta, dy, *, align_corners=True, deterministic=False, need_dx=True, need_dtheta=True, out=None):
    N, C, D, H, W = x.shape
    Do, Ho, Wo = dy.shape[2:]
    if out is not None:
        dx, dth = out
    else:
        dx = torch.empty_like(x) if need_dx else None
        dth = torch.empty((N, 3, 4), dtype=torch.float32, device=x.device) if need_dtheta else None
    o = _opts(align_corners, "zeros", "auto" if deterministic else "scatter_atomic", deterministic)
    dev = _device_of(x, dy)
    # (the stn3d query: (N, C, H, W) of the input volume with Gh = its depth, (Ho, Wo, D = Do) of the output)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_STN3D, N, C, H, W, Ho, Wo, D=Do, Gh=D, opts=o))
    _check(lib().stn3d_bwd(_ptr(x), _ptr(theta), _ptr(dy), N, C, D, H, W, Do, Ho, Wo, ctypes.byref(o), _ptr(dx),
                           _ptr(dth), _wsp(ws), nws, _stream(dev)), "stn3d_bwd")
    return dx, dth


def stn_lanczos_fwd(x, theta, Ho=None, Wo=None, *, align_corners=True, out=None):
    """Lanczos-3 STN (6 x 6 taps, zeros); CUDA tensors."""
    N, C, H, W = x.shape
    Ho = H if Ho is None else int(Ho)
    Wo = W if Wo is None else int(Wo)
    y = out if out is not None else torch.empty((N, C, Ho, Wo), dtype=torch.float32, device=x.device)
    o = _opts(align_corners)
    _check(lib().stn_lanczos_fwd(_ptr(x), _ptr(theta), N, C, H, W, Ho, Wo, ctypes.byref(o), _ptr(y),
                                 _stream(_device_of(x, y))), "stn_lanczos_fwd")
    return y


def stn_lanczos_bwd(x, theta, dy, *, align_corners=True, deterministic=False, need_dx=True, need_dtheta=True,
                    out=None):
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    if out is not None:
        dx, dth = out
    else:
        dx = torch.empty_like(x) if need_dx else None
        dth = torch.empty((N, 2, 3), dtype=torch.float32, device=x.device) if need_dtheta else None
    o = _opts(align_corners, "zeros", "auto" if deterministic else "scatter_atomic", deterministic)
    dev = _device_of(x, dy)
    ws, nws = _workspace(dev, workspace_bytes(LAYER_LANCZOS, N, C, H, W, Ho, Wo, opts=o))
    _check(lib().stn_lanczos_bwd(_ptr(x), _ptr(theta), _ptr(dy), N, C, H, W, Ho, Wo, ctypes.byref(o), _ptr(dx),
                                 _ptr(dth), _wsp(ws), nws, _stream(dev)), "stn_lanczos_bwd")
    return dx, dth
