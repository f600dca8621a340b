"""Seeded synthetic inputs for the resampling layers (shared by tests, bench, oracle runs).

This module holds the INPUT RECIPE only — distributions, shapes and seeds —
and none of the method's arithmetic (no sampling, slicing or adjoints).  Both
the CUDA path and the fp64 oracle consume what it produces; neither is
imported here.

Recipe:
  * per-sample seeding: sample n of config ``cfg`` draws tensor kind k from a
    generator seeded with ``((1000*cfg + n) * 16 + k)``, so a batch shard on any
    rank regenerates exactly the samples of the unsharded batch;
  * STN ("512x512, 16 channels, batch 4"): X ~ N(0,1) iid
    (or a smooth sum of 8 sinusoids), theta = s R(a) [[1,h],[0,1]] | t with
    a ~ U(-30deg, 30deg), s ~ U(0.8, 1.2), h ~ U(-0.05, 0.05), t ~ U(-0.2, 0.2)^2,
    dY ~ N(0,1);
  * warp (FlowNet 2.0): X ~ U(0,1); "smooth" flow = a coarse
    (H/32+1)x(W/32+1) N(0, 8^2) px field, bilinearly upsampled, plus iid
    N(0, 0.5^2) px; "stress" flow = iid U(-32, 32) px; dY ~ N(0,1);
  * bslice (HDRNet): grid = identity affine + N(0, 0.1^2)
    (or iid N(0,1)); guide ~ U(0,1) iid (or a smooth luminance field);
    X ~ U(0,1); dY ~ N(0,1).

Generation runs in float64 on the CPU and is cast to float32 (canonical, used
by every parity test), or — for the large bench workloads only — in float32
with a CUDA generator (``device='cuda'``), documented as such in bench output.
"""
from __future__ import annotations

import math

import torch

# tensor-kind ids for the per-sample seed
_X, _THETA, _DY, _FLOW, _GRID, _GUIDE, _FLOW2 = range(7)


def _gen(cfg: int, n: int, kind: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(((1000 * int(cfg) + int(n)) * 16 + kind) & 0x7FFFFFFFFFFFFFFF)
    return g


def _dtype(device):
    return torch.float64 if torch.device(device).type == "cpu" else torch.float32


def _per_sample(N, shape, cfg, kind, device, draw, n0=0):
    """Stack per-sample draws; draw(gen, shape, dtype) -> tensor."""
    dt = _dtype(device)
    out = [draw(_gen(cfg, n0 + n, kind, device), shape, dt) for n in range(N)]
    return torch.stack(out).to(torch.float32)


def _normal(g, shape, dt, std=1.0, mean=0.0):
    return torch.randn(shape, generator=g, dtype=dt, device=g.device) * std + mean


def _uniform(g, shape, dt, lo=0.0, hi=1.0):
    return torch.rand(shape, generator=g, dtype=dt, device=g.device) * (hi - lo) + lo


def _sinusoids(g, shape, dt, k=8, lam_lo=16.0, lam_hi=128.0):
    """Smooth field: sum of k random plane waves, wavelengths U(lam_lo, lam_hi) px."""
    C, H, W = shape
    dev = g.device
    yy = torch.arange(H, dtype=dt, device=dev).view(H, 1)
    xx = torch.arange(W, dtype=dt, device=dev).view(1, W)
    out = torch.zeros(shape, dtype=dt, device=dev)
    for c in range(C):
        for _ in range(k):
            p = torch.rand(4, generator=g, dtype=dt, device=dev)
            lam = lam_lo + (lam_hi - lam_lo) * p[0]
            ang = 2 * math.pi * p[1]
            ph = 2 * math.pi * p[2]
            amp = 0.5 + p[3]
            out[c] += amp * torch.sin(2 * math.pi / lam * (torch.cos(ang) * xx + torch.sin(ang) * yy) + ph)
    return out / math.sqrt(k)


# ----------------------------------------------------------------------------- STN
def stn_theta(N, cfg, device="cpu", kind="random", n0=0):
    """Per-sample affine theta (N x 2 x 3)."""
    if kind == "identity":
        t = torch.tensor([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]], dtype=torch.float64)
        return t.expand(N, 2, 3).contiguous().to(torch.float32).to(device)

    def draw(g, shape, dt):
        p = torch.rand(6, generator=g, dtype=dt, device=g.device)
        a = (p[0] * 2 - 1) * (math.pi / 6)
        s = 0.8 + 0.4 * p[1]
        h = (p[2] * 2 - 1) * 0.05
        tx = (p[3] * 2 - 1) * 0.2
        ty = (p[4] * 2 - 1) * 0.2
        c, sn = torch.cos(a), torch.sin(a)
        m00, m01 = s * c, s * (c * h - sn)
        m10, m11 = s * sn, s * (sn * h + c)
        return torch.stack([torch.stack([m00, m01, tx]), torch.stack([m10, m11, ty])])

    return _per_sample(N, None, cfg, _THETA, device, draw, n0)


def stn_inputs(N, C, H, W, Ho=None, Wo=None, *, cfg=2, device="cpu", smooth=False,
               theta_kind="random", n0=0):
    Ho = H if Ho is None else Ho
    Wo = W if Wo is None else Wo
    if smooth:
        x = _per_sample(N, (C, H, W), cfg, _X, device, _sinusoids, n0)
    else:
        x = _per_sample(N, (C, H, W), cfg, _X, device, _normal, n0)
    theta = stn_theta(N, cfg, device, theta_kind, n0)
    dy = _per_sample(N, (C, Ho, Wo), cfg, _DY, device, _normal, n0)
    return {"x": x, "theta": theta, "dy": dy}


# ----------------------------------------------------------------------------- warp
def _smooth_flow(g, shape, dt):
    _, H, W = shape
    hc, wc = H // 32 + 1, W // 32 + 1
    coarse = torch.randn((1, 2, hc, wc), generator=g, dtype=dt, device=g.device) * 8.0
    up = torch.nn.functional.interpolate(coarse, size=(H, W), mode="bilinear", align_corners=True)[0]
    return up + torch.randn((2, H, W), generator=g, dtype=dt, device=g.device) * 0.5


def _stress_flow(g, shape, dt):
    return _uniform(g, shape, dt, -32.0, 32.0)


def warp_inputs(N, C, H, W, *, cfg=3, device="cpu", flow="smooth", n0=0):
    x = _per_sample(N, (C, H, W), cfg, _X, device, _uniform, n0)
    if flow == "smooth":
        f = _per_sample(N, (2, H, W), cfg, _FLOW, device, _smooth_flow, n0)
    elif flow == "stress":
        f = _per_sample(N, (2, H, W), cfg, _FLOW2, device, _stress_flow, n0)
    elif flow == "zero":
        f = torch.zeros((N, 2, H, W), dtype=torch.float32, device=device)
    else:
        raise ValueError(flow)
    dy = _per_sample(N, (C, H, W), cfg, _DY, device, _normal, n0)
    return {"x": x, "flow": f, "dy": dy}


# ----------------------------------------------------------------------------- bslice
def _identity_grid(g, shape, dt, std=0.1):
    _, D, Gh, Gw = shape
    base = torch.zeros(shape, dtype=dt, device=g.device)
    for o in range(3):
        base[4 * o + o] = 1.0
    return base + torch.randn(shape, generator=g, dtype=dt, device=g.device) * std


def _smooth_guide(g, shape, dt):
    H, W = shape
    s = _sinusoids(g, (1, H, W), dt, k=8, lam_lo=32.0, lam_hi=256.0)[0]
    return 0.5 + 0.35 * torch.tanh(s)


def bslice_inputs(N, H, W, D=8, Gh=16, Gw=16, *, cfg=4, device="cpu", grid="identity",
                  guide="uniform", n0=0):
    gshape = (12, D, Gh, Gw)
    if grid == "identity":
        gr = _per_sample(N, gshape, cfg, _GRID, device, _identity_grid, n0)
    elif grid == "iid":
        gr = _per_sample(N, gshape, cfg, _GRID, device, _normal, n0)
    else:
        raise ValueError(grid)
    if guide == "uniform":
        gd = _per_sample(N, (H, W), cfg, _GUIDE, device, _uniform, n0)
    elif guide == "smooth":
        gd = _per_sample(N, (H, W), cfg, _GUIDE, device, _smooth_guide, n0)
    elif guide == "wide":  # outside [0,1]: exercises clamped z planes
        gd = _per_sample(N, (H, W), cfg, _GUIDE, device,
                         lambda g, s, dt: _uniform(g, s, dt, -0.2, 1.2), n0)
    else:
        raise ValueError(guide)
    x = _per_sample(N, (3, H, W), cfg, _X, device, _uniform, n0)
    dy = _per_sample(N, (3, H, W), cfg, _DY, device, _normal, n0)
    return {"grid": gr, "guide": gd, "x": x, "dy": dy}
