"""fp64 CPU oracle for the resampling layers (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1904_12228_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c``; this module only marshals
numpy float64 arrays through ctypes.

Every function here follows the definitions cited in ``oracle.c``
(PAPER.md:21-42 layers; PAPER.md:684, 2239-2241 VJP semantics; PAPER.md:700-707
naive scatter adjoint).  Pins: ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int
        lib.oracle_stn_fwd.argtypes = [P, P, I, I, I, I, I, I, I, I, P]
        lib.oracle_stn_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, I, P, P]
        lib.oracle_warp_fwd.argtypes = [P, P, I, I, I, I, I, P]
        lib.oracle_warp_bwd.argtypes = [P, P, P, I, I, I, I, I, P, P]
        lib.oracle_bslice_fwd.argtypes = [P, P, P, I, I, I, I, I, I, P]
        lib.oracle_bslice_bwd.argtypes = [P, P, P, P, I, I, I, I, I, I, P, P, P]
        lib.oracle_conv_fwd.argtypes = [P, P, I, I, I, I, I, I, I, P]
        lib.oracle_conv_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, P, P]
        lib.oracle_convloss_grad.argtypes = [P, P, P, I, I, I, I, I, P]
        lib.oracle_upsample4_fwd.argtypes = [P, I, I, I, I, P]
        lib.oracle_upsample4_bwd.argtypes = [P, I, I, I, I, P]
        lib.oracle_stn_bicubic_fwd.argtypes = [P, P, I, I, I, I, I, I, I, P]
        lib.oracle_stn_bicubic_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, P, P]
        lib.oracle_stn3d_fwd.argtypes = [P, P, I, I, I, I, I, I, I, I, I, P]
        lib.oracle_stn3d_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, I, I, P, P]
        lib.oracle_stn_kinks.argtypes = [P, I, I, I, I, I, I, ctypes.c_double]
        lib.oracle_stn_kinks.restype = ctypes.c_long
        lib.oracle_warp_kinks.argtypes = [P, I, I, I, ctypes.c_double]
        lib.oracle_warp_kinks.restype = ctypes.c_long
        lib.oracle_bslice_kinks.argtypes = [P, I, I, I, I, ctypes.c_double]
        lib.oracle_bslice_kinks.restype = ctypes.c_long
        lib.oracle_stn_lanczos_fwd.argtypes = [P, P, I, I, I, I, I, I, I, P]
        lib.oracle_stn_lanczos_bwd.argtypes = [P, P, P, I, I, I, I, I, I, I, P, P]
        lib.oracle_lanczos3.argtypes = [ctypes.c_double]
        lib.oracle_lanczos3.restype = ctypes.c_double
        lib.oracle_dlanczos3.argtypes = [ctypes.c_double]
        lib.oracle_dlanczos3.restype = ctypes.c_double
        lib.oracle_set_threads.argtypes = [I]
        lib.oracle_get_threads.restype = I
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


# ----------------------------------------------------------------------------- STN
def stn_fwd(x, theta, Ho=None, Wo=None, align_corners=True, border=False):
    x, theta = _f64(x), _f64(theta)
    N, C, H, W = x.shape
    Ho = H if Ho is None else Ho
    Wo = W if Wo is None else Wo
    y = np.empty((N, C, Ho, Wo), np.float64)
    _load().oracle_stn_fwd(_p(x), _p(theta), N, C, H, W, Ho, Wo, int(align_corners),
                           int(border), _p(y))
    return y


def stn_bwd(x, theta, dy, align_corners=True, border=False, need_dx=True, need_dtheta=True):
    x, theta, dy = _f64(x), _f64(theta), _f64(dy)
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    dx = np.empty_like(x) if need_dx else None
    dth = np.empty((N, 2, 3), np.float64) if need_dtheta else None
    _load().oracle_stn_bwd(_p(x), _p(theta), _p(dy), N, C, H, W, Ho, Wo, int(align_corners),
                           int(border), _p(dx), _p(dth))
    return dx, dth


# ----------------------------------------------------------------------------- warp
def warp_fwd(x, flow, border=False):
    x, flow = _f64(x), _f64(flow)
    N, C, H, W = x.shape
    y = np.empty_like(x)
    _load().oracle_warp_fwd(_p(x), _p(flow), N, C, H, W, int(border), _p(y))
    return y


def warp_bwd(x, flow, dy, border=False, need_dx=True, need_dflow=True):
    x, flow, dy = _f64(x), _f64(flow), _f64(dy)
    N, C, H, W = x.shape
    dx = np.empty_like(x) if need_dx else None
    df = np.empty_like(flow) if need_dflow else None
    _load().oracle_warp_bwd(_p(x), _p(flow), _p(dy), N, C, H, W, int(border), _p(dx), _p(df))
    return dx, df


# ----------------------------------------------------------------------------- bslice
def bslice_fwd(grid, guide, x):
    grid, guide, x = _f64(grid), _f64(guide), _f64(x)
    N, Q, D, Gh, Gw = grid.shape
    assert Q == 12 and x.shape[1] == 3
    H, W = guide.shape[1:]
    y = np.empty_like(x)
    _load().oracle_bslice_fwd(_p(grid), _p(guide), _p(x), N, H, W, D, Gh, Gw, _p(y))
    return y


def bslice_bwd(grid, guide, x, dy, need_dgrid=True, need_dguide=True, need_dx=True):
    grid, guide, x, dy = _f64(grid), _f64(guide), _f64(x), _f64(dy)
    N, Q, D, Gh, Gw = grid.shape
    H, W = guide.shape[1:]
    dgrid = np.empty_like(grid) if need_dgrid else None
    dguide = np.empty_like(guide) if need_dguide else None
    dx = np.empty_like(x) if need_dx else None
    _load().oracle_bslice_bwd(_p(grid), _p(guide), _p(x), _p(dy), N, H, W, D, Gh, Gw,
                              _p(dgrid), _p(dguide), _p(dx))
    return dgrid, dguide, dx


# ----------------------------------------------------------------------------- conv (§8(f) f1)
def conv_fwd(x, k):
    """y = sum_{ci,ry,rx} x[n,ci,y-ry+kh//2,x-rx+kw//2] k[co,ci,ry,rx] (PAPER.md:703-707, 2-D)."""
    x, k = _f64(x), _f64(k)
    N, Ci, H, W = x.shape
    Co, Ci2, kh, kw = k.shape
    assert Ci2 == Ci
    y = np.empty((N, Co, H, W), np.float64)
    _load().oracle_conv_fwd(_p(x), _p(k), N, Ci, Co, H, W, kh, kw, _p(y))
    return y


def conv_bwd(x, k, dy, need_dx=True, need_dk=True):
    """dx by the naive scatter, dk by its definition."""
    x, k, dy = _f64(x), _f64(k), _f64(dy)
    N, Ci, H, W = x.shape
    Co, _, kh, kw = k.shape
    dx = np.empty_like(x) if need_dx else None
    dk = np.empty_like(k) if need_dk else None
    _load().oracle_conv_bwd(_p(x), _p(k), _p(dy), N, Ci, Co, H, W, kh, kw, _p(dx), _p(dk))
    return dx, dk


# ----------------------------------------------------------------------------- §8(f) f4
def convloss_grad(inp, k, target):
    """d_in of loss = sum (conv(in, k) - target)^2, single channel."""
    inp, k, target = _f64(inp), _f64(k), _f64(target)
    N, H, W = inp.shape
    kh, kw = k.shape
    d = np.empty_like(inp)
    _load().oracle_convloss_grad(_p(inp), _p(k), _p(target), N, H, W, kh, kw, _p(d))
    return d


def upsample4_fwd(x):
    x = _f64(x)
    N, C, H, W = x.shape
    y = np.empty((N, C, 4 * H, 4 * W), np.float64)
    _load().oracle_upsample4_fwd(_p(x), N, C, H, W, _p(y))
    return y


def upsample4_bwd(dy):
    dy = _f64(dy)
    N, C, Ho, Wo = dy.shape
    dx = np.empty((N, C, Ho // 4, Wo // 4), np.float64)
    _load().oracle_upsample4_bwd(_p(dy), N, C, Ho // 4, Wo // 4, _p(dx))
    return dx


# ----------------------------------------------------------------------------- §8(f) f3
def stn_bicubic_fwd(x, theta, Ho=None, Wo=None, align_corners=True):
    x, theta = _f64(x), _f64(theta)
    N, C, H, W = x.shape
    Ho = H if Ho is None else Ho
    Wo = W if Wo is None else Wo
    y = np.empty((N, C, Ho, Wo), np.float64)
    _load().oracle_stn_bicubic_fwd(_p(x), _p(theta), N, C, H, W, Ho, Wo, int(align_corners), _p(y))
    return y


def stn_bicubic_bwd(x, theta, dy, align_corners=True):
    x, theta, dy = _f64(x), _f64(theta), _f64(dy)
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    dx, dth = np.empty_like(x), np.empty((N, 2, 3), np.float64)
    _load().oracle_stn_bicubic_bwd(_p(x), _p(theta), _p(dy), N, C, H, W, Ho, Wo, int(align_corners), _p(dx),
                                   _p(dth))
    return dx, dth


def stn3d_fwd(x, theta, out_size=None, align_corners=True):
    x, theta = _f64(x), _f64(theta)
    N, C, D, H, W = x.shape
    Do, Ho, Wo = (D, H, W) if out_size is None else out_size
    y = np.empty((N, C, Do, Ho, Wo), np.float64)
    _load().oracle_stn3d_fwd(_p(x), _p(theta), N, C, D, H, W, Do, Ho, Wo, int(align_corners), _p(y))
    return y


def stn3d_bwd(x, theta, dy, align_corners=True):
    x, theta, dy = _f64(x), _f64(theta), _f64(dy)
    N, C, D, H, W = x.shape
    Do, Ho, Wo = dy.shape[2:]
    dx, dth = np.empty_like(x), np.empty((N, 3, 4), np.float64)
    _load().oracle_stn3d_bwd(_p(x), _p(theta), _p(dy), N, C, D, H, W, Do, Ho, Wo, int(align_corners), _p(dx),
                             _p(dth))
    return dx, dth


# ----------------------------------------------------------------------------- diagnostics
def stn_kinks(theta, H, W, Ho=None, Wo=None, align_corners=True, tol=1e-6):
    """Sample coordinates (per axis) within tol px of an integer (SURVEY 8(c) diagnostic)."""
    theta = _f64(theta)
    Ho = H if Ho is None else Ho
    Wo = W if Wo is None else Wo
    return int(_load().oracle_stn_kinks(_p(theta), theta.shape[0], H, W, Ho, Wo, int(align_corners), tol))


def warp_kinks(flow, tol=1e-6):
    flow = _f64(flow)
    N, _, H, W = flow.shape
    return int(_load().oracle_warp_kinks(_p(flow), N, H, W, tol))


def bslice_kinks(guide, D, tol=1e-6):
    guide = _f64(guide)
    N, H, W = guide.shape
    return int(_load().oracle_bslice_kinks(_p(guide), N, H, W, D, tol))


def lanczos3(x):
    return float(_load().oracle_lanczos3(float(x)))


def dlanczos3(x):
    return float(_load().oracle_dlanczos3(float(x)))


def stn_lanczos_fwd(x, theta, Ho=None, Wo=None, align_corners=True):
    x, theta = _f64(x), _f64(theta)
    N, C, H, W = x.shape
    Ho = H if Ho is None else Ho
    Wo = W if Wo is None else Wo
    y = np.empty((N, C, Ho, Wo), np.float64)
    _load().oracle_stn_lanczos_fwd(_p(x), _p(theta), N, C, H, W, Ho, Wo, int(align_corners), _p(y))
    return y


def stn_lanczos_bwd(x, theta, dy, align_corners=True):
    x, theta, dy = _f64(x), _f64(theta), _f64(dy)
    N, C, H, W = x.shape
    Ho, Wo = dy.shape[2:]
    dx, dth = np.empty_like(x), np.empty((N, 2, 3), np.float64)
    _load().oracle_stn_lanczos_bwd(_p(x), _p(theta), _p(dy), N, C, H, W, Ho, Wo, int(align_corners), _p(dx),
                                   _p(dth))
    return dx, dth
