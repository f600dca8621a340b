"""CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerance (tests/_tol.py): |g - r| <= rtol |r| + atol max(1, rms(r)); forward
rtol 1e-5, gradients rtol 1e-4, atol 1e-6 (BASELINE.json north_star).
Sizes: configs[0] (STN 1x3x16x16), ragged multi-tile shapes, and the paper
shapes of configs[1..3] in full; configs[4] (batch 64 @ 1024^2) is run in the
bench launch configuration and compared on sampled whole samples (every
sample is independent).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1904_12228_b200 import rsgrad
from _tol import assert_close, compare  # noqa: E402

pytestmark = pytest.mark.gpu


def _cuda(d, dev):
    return {k: v.to(dev).contiguous() for k, v in d.items()}


def _np(t):
    return t.detach().cpu().double().numpy()


# ============================================================================ STN
STN_SHAPES = [
    (1, 3, 16, 16, 16, 16),     # configs[0]
    (2, 5, 37, 53, 41, 29),     # ragged, several tiles, Ho != H
    (3, 16, 64, 96, 64, 96),
    (1, 1, 2, 2, 2, 2),         # minimum for align_corners=1
]


@pytest.mark.parametrize("shape", STN_SHAPES)
@pytest.mark.parametrize("ac", [True, False])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_stn_parity(cuda_device, shape, ac, padding):
    N, C, H, W, Ho, Wo = shape
    inp = synth.stn_inputs(N, C, H, W, Ho, Wo, cfg=1)
    g = _cuda(inp, cuda_device)
    y = rsgrad.stn_fwd(g["x"], g["theta"], Ho, Wo, align_corners=ac, padding=padding)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], align_corners=ac, padding=padding)
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    border = padding == "border"
    ry = oracle.stn_fwd(x, th, Ho, Wo, ac, border)
    rdx, rdth = oracle.stn_bwd(x, th, dy, ac, border)
    assert_close(_np(y), ry, "fwd", "y")
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


@pytest.mark.parametrize("algo", ["gather", "scatter_priv", "scatter_atomic"])
def test_stn_algos_agree_with_oracle(cuda_device, algo):
    inp = synth.stn_inputs(2, 8, 48, 40, cfg=1)
    g = _cuda(inp, cuda_device)
    dx, _ = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], algo=algo, need_dtheta=False)
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")))
    assert_close(_np(dx), rdx, "grad", f"dx[{algo}]")
    dx2, dth2 = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], algo=algo)
    assert_close(_np(dx2), rdx, "grad", f"dx[{algo}] with dtheta")
    assert_close(_np(dth2), rdth, "grad", f"dtheta[{algo}]")


@pytest.mark.parametrize("shape", [(2, 5, 37, 53, 41, 29), (1, 16, 64, 96, 64, 96), (2, 3, 20, 24, 20, 24)])
@pytest.mark.parametrize("padding", ["zeros", "border"])
@pytest.mark.parametrize("ac", [True, False])
def test_stn_scatter_priv_parity(cuda_device, shape, padding, ac):
    """SCATTER_PRIV: d_input via the block-private footprint accumulator, every sample."""
    N, C, H, W, Ho, Wo = shape
    inp = synth.stn_inputs(N, C, H, W, Ho, Wo, cfg=1)
    g = _cuda(inp, cuda_device)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], align_corners=ac, padding=padding,
                             algo="scatter_priv")
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")), ac,
                               padding == "border")
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


def test_stn_fallback_samples_priv_and_atomic(cuda_device):
    """Fallback samples (singular / huge preimage) inside an AUTO batch: privatised dX,
    alone (need_dtheta=False) and with d_theta; and the SCATTER_ATOMIC route."""
    inp = synth.stn_inputs(4, 6, 40, 44, cfg=1)
    inp["theta"][1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])
    inp["theta"][3] = torch.tensor([[0.02, 0.0, 0.1], [0.0, 0.03, 0.0]])
    g = _cuda(inp, cuda_device)
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")))
    dx, _ = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], need_dtheta=False)
    assert_close(_np(dx), rdx, "grad", "dx (AUTO, no dtheta)")
    for algo in ("auto", "scatter_atomic"):
        dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], algo=algo)
        assert_close(_np(dx), rdx, "grad", f"dx [{algo}]")
        assert_close(_np(dth), rdth, "grad", f"dtheta [{algo}]")


@pytest.mark.parametrize("scale", [0.79, 0.85])
def test_stn_lean_near_record_cap(cuda_device, scale):
    """Zoomed-in affine maps (scale < 1: ~1/s^2 output pixels per input cell) fill the lean
    kernel's per-tile record and hit-list buffers close to their caps (2304 records) at
    every rotation; d_input is still the gather (no fallback) and matches the oracle."""
    import math
    N = 4
    inp = synth.stn_inputs(N, 4, 96, 128, cfg=1)
    for n in range(N):
        a = math.radians(15.0 * n)
        inp["theta"][n] = torch.tensor([[scale * math.cos(a), -scale * math.sin(a), 0.05],
                                        [scale * math.sin(a), scale * math.cos(a), -0.03]])
    g = _cuda(inp, cuda_device)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], deterministic=True)
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    rdx, rdth = oracle.stn_bwd(x, th, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


@pytest.mark.parametrize("groups", ["1", "2", "4"])
@pytest.mark.parametrize("flow", ["smooth", "stress"])
def test_warp_fwd_pixel_groups(cuda_device, monkeypatch, groups, flow):
    """warp_fwd with 1, 2 or 4 pixel pairs per thread (the pipelined kernel prefetches the
    next pair's flow), ragged sizes so the last block's groups run past the image."""
    monkeypatch.setenv("RSGRAD_WARP_FWD_G", groups)
    inp = synth.warp_inputs(3, 3, 37, 101, cfg=1, flow=flow)
    g = _cuda(inp, cuda_device)
    y = rsgrad.warp_fwd(g["x"], g["flow"])
    assert_close(_np(y), oracle.warp_fwd(inp["x"].double().numpy(), inp["flow"].double().numpy()), "fwd", "y")


def test_stn_bwd_three_launches(cuda_device, monkeypatch):
    """The lean backward path runs as three launches (lean d_input with its own sample
    classification and coordinates, d_theta tiles, finalize + fallback scatter) and agrees
    bitwise with the path that prepares tables and classes in a separate kernel
    (RSGRAD_STN_PREP); with fallback samples (singular / huge preimage) both match the oracle."""
    inp = synth.stn_inputs(3, 8, 64, 96, cfg=1)
    g = _cuda(inp, cuda_device)
    rsgrad.launch_count(reset=True)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    assert rsgrad.launch_count() == 3
    monkeypatch.setenv("RSGRAD_STN_PREP", "1")
    dx2, dth2 = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    assert torch.equal(dx, dx2) and torch.equal(dth, dth2)
    monkeypatch.delenv("RSGRAD_STN_PREP")
    inp["theta"][1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])   # det = 0
    inp["theta"][2] = torch.tensor([[0.02, 0.0, 0.1], [0.0, 0.03, 0.0]])  # huge preimage
    g = _cuda(inp, cuda_device)
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    rdx, rdth = oracle.stn_bwd(x, th, dy)
    for need_dtheta in (True, False):
        dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], need_dtheta=need_dtheta)
        assert_close(_np(dx), rdx, "grad", "dx")
        if need_dtheta:
            assert_close(_np(dth), rdth, "grad", "dtheta")
    _, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], need_dx=False)
    assert_close(_np(dth), rdth, "grad", "dtheta only")


@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_stn_high_fan_in_fallback(cuda_device, padding):
    """AUTO fallback samples whose map piles many output pixels onto one input cell (a
    near-singular map, strong zoom-out: thousands of taps per element; 2x zoom-out under
    border padding: clamped taps on the edges) stay within T: the scatter pre-sums each
    warp's runs of equal tap address before its reds."""
    inp = synth.stn_inputs(4, 4, 64, 96, cfg=1)
    inp["theta"][0] = torch.tensor([[0.02, 0.0, 0.1], [0.0, 0.03, 0.0]])
    inp["theta"][1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])
    inp["theta"][2] = torch.tensor([[2.0, 0.0, 0.0], [0.0, 2.0, 0.0]])
    inp["theta"][3] = torch.tensor([[0.05, 0.01, -0.3], [-0.02, 0.04, 0.2]])
    g = _cuda(inp, cuda_device)
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    rdx, rdth = oracle.stn_bwd(x, th, dy, True, padding == "border")
    for _ in range(3):
        dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], padding=padding)
        assert_close(_np(dx), rdx, "grad", "dx")
        assert_close(_np(dth), rdth, "grad", "dtheta")


@pytest.mark.parametrize("fork", ["0", "100000"])
def test_stn_bwd_fork(cuda_device, monkeypatch, fork):
    """The d_theta tiles on the library side stream beside the lean d_input kernel, or
    after it on the caller's stream: both match the oracle and agree bitwise."""
    monkeypatch.setenv("RSGRAD_STN_FORK", fork)
    inp = synth.stn_inputs(3, 16, 80, 96, cfg=1)
    g = _cuda(inp, cuda_device)
    y = rsgrad.stn_fwd(g["x"], g["theta"])
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    assert_close(_np(y), oracle.stn_fwd(x, th), "fwd", "y")
    rdx, rdth = oracle.stn_bwd(x, th, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")
    monkeypatch.setenv("RSGRAD_STN_FORK", "0" if fork != "0" else "100000")
    dx2, dth2 = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    assert torch.equal(dx, dx2) and torch.equal(dth, dth2)


def test_stn_singular_theta_falls_back(cuda_device):
    """A rank-deficient theta has no bounded preimage: AUTO must take the atomic scatter."""
    inp = synth.stn_inputs(3, 4, 20, 24, cfg=1)
    inp["theta"][1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])  # det = 0
    inp["theta"][2] = torch.tensor([[0.01, 0.0, 0.0], [0.0, 0.01, 0.0]])  # huge preimage
    g = _cuda(inp, cuda_device)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")))
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_stn_deterministic_every_sample(cuda_device, padding):
    """deterministic=1 is bitwise reproducible for EVERY sample: regular samples take the
    cell-owner gather, fallback samples (singular theta, huge preimage) and border padding
    the fixed-point integer scatter (det.cuh) instead of fp32 atomics; all within T."""
    inp = synth.stn_inputs(4, 6, 40, 44, cfg=1)
    inp["theta"][1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.2]])   # det = 0
    inp["theta"][3] = torch.tensor([[0.02, 0.0, 0.1], [0.0, 0.03, 0.0]])  # huge preimage
    g = _cuda(inp, cuda_device)
    runs = [rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], padding=padding, deterministic=True) for _ in range(3)]
    for r in runs[1:]:
        assert torch.equal(r[0], runs[0][0]) and torch.equal(r[1], runs[0][1])
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")), True, padding == "border")
    assert_close(_np(runs[0][0]), rdx, "grad", "dx")
    assert_close(_np(runs[0][1]), rdth, "grad", "dtheta")
    # without dtheta (the fallback list still drives the scatter)
    dx, _ = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], padding=padding, deterministic=True, need_dtheta=False)
    assert torch.equal(dx, runs[0][0])


@pytest.mark.parametrize("flow", ["smooth", "stress", "collapse"])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_deterministic(cuda_device, flow, padding):
    """warp_bwd deterministic=1: d_input by the fixed-point scatter (bitwise reproducible,
    |error| <= fan-in * 2^-(S+1), so also the collapsing flow is well inside T), d_flow by
    the strip kernel's gather (no atomics)."""
    N, C, H, W = 2, 3, 70, 100
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow="stress" if flow == "collapse" else flow)
    if flow == "collapse":
        inp["flow"] = _collapse_flow(N, H, W)
    g = _cuda(inp, cuda_device)
    a = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding, deterministic=True)
    b = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding, deterministic=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    rdx, rdf = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")), padding == "border")
    rep = assert_close(_np(a[0]), rdx, "grad", "dx")
    # fixed point: the accumulation adds ~1e-11; what remains is the fp32 tap weights
    # (~1e-7 relative per term), as in every other path -- far inside T even for the
    # collapsing flow's ~1300 terms per element
    assert rep["max_ratio"] < 0.25, rep
    assert_close(_np(a[1]), rdf, "grad", "dflow")
    dx_only, none = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding, deterministic=True,
                                    need_dflow=False)
    assert none is None and torch.equal(dx_only, a[0])


def test_warp_deterministic_nonfinite_and_zero(cuda_device):
    """Fixed-point edge cases: an all-zero dY (scale exponent 0) gives exactly 0; a
    non-finite dY makes that sample's dX NaN (the fp32 path would propagate it too)
    and leaves the other sample exact."""
    inp = synth.warp_inputs(2, 2, 20, 33, cfg=1)
    inp["dy"][0].zero_()
    g = _cuda(inp, cuda_device)
    dx, _ = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], deterministic=True)
    assert torch.count_nonzero(dx[0]) == 0
    rdx, _ = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")))
    assert_close(_np(dx[1]), rdx[1], "grad", "dx sample 1")
    bad = g["dy"].clone()
    bad[0, 0, 3, 4] = float("inf")
    dxb, _ = rsgrad.warp_bwd(g["x"], g["flow"], bad, deterministic=True)
    assert torch.isnan(dxb[0]).all() and torch.equal(dxb[1], dx[1])


def test_stn_identity_and_quarter_pixel(cuda_device):
    N, C, H, W = 2, 3, 32, 48
    inp = synth.stn_inputs(N, C, H, W, cfg=1, theta_kind="identity")
    g = _cuda(inp, cuda_device)
    y = rsgrad.stn_fwd(g["x"], g["theta"])
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    assert_close(_np(y), x, "fwd", "identity y = x")
    assert_close(_np(dx), dy, "grad", "identity dx = dy")
    # the fp64 coordinates are bit-identical to the oracle's, so even the
    # kink-sensitive d_theta at identity theta matches it (P1)
    assert_close(_np(dth), oracle.stn_bwd(x, th, dy)[1], "grad", "identity dtheta")
    q = torch.tensor([[1.0, 0.0, 0.5 / (W - 1)], [0.0, 1.0, 0.5 / (H - 1)]]).expand(N, 2, 3).contiguous()
    dxq, dthq = rsgrad.stn_bwd(g["x"], q.to(cuda_device), g["dy"])
    rq = oracle.stn_bwd(x, q.double().numpy(), dy)
    assert_close(_np(dxq), rq[0], "grad", "quarter dx")
    assert_close(_np(dthq), rq[1], "grad", "quarter dtheta")


def test_stn_gather_is_deterministic(cuda_device):
    inp = synth.stn_inputs(2, 16, 64, 64, cfg=1)
    g = _cuda(inp, cuda_device)
    a = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], deterministic=True)
    b = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], deterministic=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_stn_paper_shape_full(cuda_device):
    """configs[1]: STN 4 x 16 x 512 x 512, every element vs the oracle."""
    inp = synth.stn_inputs(4, 16, 512, 512, cfg=2)
    g = _cuda(inp, cuda_device)
    y = rsgrad.stn_fwd(g["x"], g["theta"])
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    assert_close(_np(y), oracle.stn_fwd(x, th), "fwd", "y")
    rdx, rdth = oracle.stn_bwd(x, th, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


# ============================================================================ warp
@pytest.mark.parametrize("shape", [(1, 3, 16, 16), (2, 3, 37, 61), (1, 7, 5, 130), (1, 1, 1, 1),
                                   (2, 3, 37, 64), (1, 5, 9, 132), (1, 2, 3, 4)])
@pytest.mark.parametrize("flow", ["smooth", "stress", "zero"])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_parity(cuda_device, shape, flow, padding):
    N, C, H, W = shape
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow=flow)
    g = _cuda(inp, cuda_device)
    y = rsgrad.warp_fwd(g["x"], g["flow"], padding=padding)
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding)
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    border = padding == "border"
    assert_close(_np(y), oracle.warp_fwd(x, fl, border), "fwd", "y")
    rdx, rdf = oracle.warp_bwd(x, fl, dy, border)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


@pytest.mark.parametrize("shape", [(1, 3, 16, 16), (2, 3, 37, 61), (1, 7, 5, 130), (1, 20, 33, 40)])
@pytest.mark.parametrize("flow", ["smooth", "stress", "zero"])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_scatter_priv_parity(cuda_device, shape, flow, padding):
    """SCATTER_PRIV: block-private footprint accumulation, flushed with one red per touched
    element (stress flows overflow the footprint and take per-tap reds inside the tile)."""
    N, C, H, W = shape
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow=flow)
    g = _cuda(inp, cuda_device)
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding, algo="scatter_priv")
    rdx, rdf = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")), padding == "border")
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


@pytest.mark.parametrize("flow", ["smooth", "stress"])
def test_warp_paper_shape_full(cuda_device, flow):
    """configs[2]: warp 8 x 3 x 384 x 512, every element vs the oracle."""
    inp = synth.warp_inputs(8, 3, 384, 512, cfg=3, flow=flow)
    g = _cuda(inp, cuda_device)
    y = rsgrad.warp_fwd(g["x"], g["flow"])
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"])
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    assert_close(_np(y), oracle.warp_fwd(x, fl), "fwd", "y")
    rdx, rdf = oracle.warp_bwd(x, fl, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


# ============================================================================ bslice
BS_SHAPES = [
    (1, 64, 64, 8, 4, 4),        # tiled path, 16 px cells
    (2, 100, 130, 8, 6, 7),      # ragged tiles, non-integer cell size
    (1, 300, 260, 5, 3, 2),      # large dual cells -> sub-tiles
    (1, 16, 16, 8, 16, 16),      # cells < 8 px -> generic atomic path
    (1, 9, 11, 3, 1, 1),         # single cell
    (1, 1, 1, 2, 1, 1),          # single pixel
]


@pytest.mark.parametrize("shape", BS_SHAPES)
@pytest.mark.parametrize("guide", ["uniform", "wide", "smooth"])
def test_bslice_parity(cuda_device, shape, guide):
    N, H, W, D, Gh, Gw = shape
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, grid="iid", guide=guide)
    g = _cuda(inp, cuda_device)
    y = rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dgr), rgr, "grad", "dgrid")


@pytest.mark.parametrize("shape", BS_SHAPES[:3] + [(2, 256, 192, 8, 4, 3), (1, 128, 128, 9, 4, 4)])
@pytest.mark.parametrize("guide", ["uniform", "smooth"])
def test_bslice_bwd_split_vs_tiled(cuda_device, monkeypatch, shape, guide):
    """Both dual-cell backward kernels (RSGRAD_BSLICE_BWD=split|tiled) match the oracle;
    their dX / d_guide share one summation order (bitwise equal), d_grid differs only
    in how the pixel sums are split (sub-tiles, lane ranges)."""
    N, H, W, D, Gh, Gw = shape
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, grid="iid", guide=guide)
    g = _cuda(inp, cuda_device)
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    res = {}
    for kern in ("split", "tiled"):
        monkeypatch.setenv("RSGRAD_BSLICE_BWD", kern)
        dgr, dgd, dx = res[kern] = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
        assert_close(_np(dx), rdx, "grad", f"dx[{kern}]")
        assert_close(_np(dgd), rgd, "grad", f"dguide[{kern}]")
        assert_close(_np(dgr), rgr, "grad", f"dgrid[{kern}]")
    assert torch.equal(res["split"][1], res["tiled"][1]) and torch.equal(res["split"][2], res["tiled"][2])
    # fixed chunk ranges and summation orders: a rerun is bitwise identical (d_grid too)
    monkeypatch.setenv("RSGRAD_BSLICE_BWD", "split")
    again = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    assert all(torch.equal(p, q) for p, q in zip(again, res["split"]))


def test_bslice_atomic_algo_and_determinism(cuda_device):
    inp = synth.bslice_inputs(2, 128, 96, 8, 8, 6, cfg=1)
    g = _cuda(inp, cuda_device)
    a = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    b = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    assert all(torch.equal(p, q) for p, q in zip(a, b))
    c = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], algo="scatter_atomic")
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr = oracle.bslice_bwd(gr, gd, x, dy)[0]
    assert_close(_np(c[0]), rgr, "grad", "dgrid atomic")


def test_bslice_constant_grid_closed_form(cuda_device):
    N, H, W, D, Gh, Gw = 2, 128, 128, 8, 8, 8
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1)
    A = torch.randn(N, 12, generator=torch.Generator().manual_seed(3))
    inp["grid"] = A.view(N, 12, 1, 1, 1).expand(N, 12, D, Gh, Gw).contiguous()
    g = _cuda(inp, cuda_device)
    _, dgd, _ = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    assert float(dgd.abs().max()) < 1e-5


def test_bslice_paper_shape_full(cuda_device):
    """configs[3]: 4 x 1024^2, grid 16x16x8, every element vs the oracle."""
    inp = synth.bslice_inputs(4, 1024, 1024, 8, 16, 16, cfg=4)
    g = _cuda(inp, cuda_device)
    y = rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dgr), rgr, "grad", "dgrid")


def test_bslice_paper_grid_32(cuda_device):
    """K4': the paper's own 1024^2 shape uses a 32x32x8 grid."""
    inp = synth.bslice_inputs(1, 1024, 1024, 8, 32, 32, cfg=4)
    g = _cuda(inp, cuda_device)
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dgr), rgr, "grad", "dgrid")
    assert_close(_np(dgd), rgd, "grad", "dguide")


def test_bslice_paper_highres_2048_g64(cuda_device):
    """the paper's high-resolution case, 2048^2 with a 64x64x8 grid
    (PAPER.md:42), one sample, every element of the forward and all gradients."""
    inp = synth.bslice_inputs(1, 2048, 2048, 8, 64, 64, cfg=4)
    g = _cuda(inp, cuda_device)
    y = rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dgr), rgr, "grad", "dgrid")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dx), rdx, "grad", "dx")


# ============================================================================ configs[4] sampled
def test_sweep_config_sampled(cuda_device):
    """configs[4]: batch 64 @ 1024^2 per layer in the bench launch configuration;
    samples {0, 41, 63} compared in full with the oracle."""
    N, H, W = 64, 1024, 1024
    pick = [0, 41, 63]
    # STN, C = 16
    inp = synth.stn_inputs(N, 16, H, W, cfg=5, device=cuda_device)
    y = rsgrad.stn_fwd(inp["x"], inp["theta"])
    dx, dth = rsgrad.stn_bwd(inp["x"], inp["theta"], inp["dy"])
    sub = {k: _np(v[pick]) for k, v in inp.items()}
    assert_close(_np(y[pick]), oracle.stn_fwd(sub["x"], sub["theta"]), "fwd", "stn y")
    rdx, rdth = oracle.stn_bwd(sub["x"], sub["theta"], sub["dy"])
    assert_close(_np(dx[pick]), rdx, "grad", "stn dx")
    assert_close(_np(dth[pick]), rdth, "grad", "stn dtheta")
    del inp, y, dx, dth
    torch.cuda.empty_cache()
    # warp, C = 3, smooth flow
    inp = synth.warp_inputs(N, 3, H, W, cfg=5, device=cuda_device)
    y = rsgrad.warp_fwd(inp["x"], inp["flow"])
    dx, df = rsgrad.warp_bwd(inp["x"], inp["flow"], inp["dy"])
    sub = {k: _np(v[pick]) for k, v in inp.items()}
    assert_close(_np(y[pick]), oracle.warp_fwd(sub["x"], sub["flow"]), "fwd", "warp y")
    rdx, rdf = oracle.warp_bwd(sub["x"], sub["flow"], sub["dy"])
    assert_close(_np(dx[pick]), rdx, "grad", "warp dx")
    assert_close(_np(df[pick]), rdf, "grad", "warp dflow")
    del inp, y, dx, df
    torch.cuda.empty_cache()
    # bslice, grid 16x16x8
    inp = synth.bslice_inputs(N, H, W, 8, 16, 16, cfg=5, device=cuda_device)
    y = rsgrad.bslice_fwd(inp["grid"], inp["guide"], inp["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(inp["grid"], inp["guide"], inp["x"], inp["dy"])
    sub = {k: _np(v[pick]) for k, v in inp.items()}
    assert_close(_np(y[pick]), oracle.bslice_fwd(sub["grid"], sub["guide"], sub["x"]), "fwd", "bs y")
    rgr, rgd, rdx = oracle.bslice_bwd(sub["grid"], sub["guide"], sub["x"], sub["dy"])
    assert_close(_np(dx[pick]), rdx, "grad", "bs dx")
    assert_close(_np(dgd[pick]), rgd, "grad", "bs dguide")
    assert_close(_np(dgr[pick]), rgr, "grad", "bs dgrid")


# ============================================================================ boundary behaviour
def test_host_pointer_path_matches_device(cuda_device):
    """CPU (pinned and pageable) tensors go through the library's staging path."""
    inp = synth.bslice_inputs(1, 64, 80, 8, 4, 5, cfg=1)
    g = _cuda(inp, cuda_device)
    ref = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    pinned = {k: v.pin_memory() for k, v in inp.items()}
    host = rsgrad.bslice_bwd(pinned["grid"], pinned["guide"], pinned["x"], pinned["dy"],
                             deterministic=True)
    for a, b in zip(ref, host):
        assert not b.is_cuda and torch.equal(a.cpu(), b)
    y_pageable = rsgrad.bslice_fwd(inp["grid"], inp["guide"], inp["x"])
    assert torch.equal(y_pageable, rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"]).cpu())


def test_autograd_wrappers(cuda_device):
    inp = synth.stn_inputs(2, 3, 24, 24, cfg=1)
    x = inp["x"].to(cuda_device).requires_grad_()
    th = inp["theta"].to(cuda_device).requires_grad_()
    y = rsgrad.SpatialTransformer.apply(x, th)
    y.backward(inp["dy"].to(cuda_device))
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")))
    assert_close(_np(x.grad), rdx, "grad", "dx")
    assert_close(_np(th.grad), rdth, "grad", "dtheta")


def test_launch_accounting(cuda_device):
    inp = _cuda(synth.warp_inputs(1, 3, 32, 32, cfg=1), cuda_device)
    rsgrad.launch_count(reset=True)
    rsgrad.warp_fwd(inp["x"], inp["flow"])
    rsgrad.warp_bwd(inp["x"], inp["flow"], inp["dy"])
    # warp_fwd: 1; warp_bwd AUTO: the strip kernel + the heavy-sample fixed-point
    # recompute (exits at once when no sample is marked heavy); the dX memset is not ours
    assert rsgrad.launch_count() == 3


def test_outputs_overwritten_not_accumulated(cuda_device):
    inp = _cuda(synth.stn_inputs(1, 4, 32, 32, cfg=1), cuda_device)
    dx = torch.full_like(inp["x"], 7.0)
    dth = torch.full((1, 2, 3), 7.0, device=cuda_device)
    rsgrad.stn_bwd(inp["x"], inp["theta"], inp["dy"], out=(dx, dth))
    ref = rsgrad.stn_bwd(inp["x"], inp["theta"], inp["dy"])
    assert torch.equal(dx, ref[0]) and torch.equal(dth, ref[1])


@pytest.mark.parametrize("variant", ["cell", "gather"])
@pytest.mark.parametrize("ac", [True, False])
def test_stn_bwd_variants(cuda_device, monkeypatch, variant, ac):
    """Both gather-form STN adjoints (cell-owner and per-pixel) match the oracle,
    including image-edge cells (x0 = -1 / y0 = -1) and a zoomed-in theta."""
    monkeypatch.setenv("RSGRAD_STN_BWD", variant)
    inp = synth.stn_inputs(3, 5, 70, 90, 66, 94, cfg=1)
    inp["theta"][2] = torch.tensor([[0.8, 0.05, 0.1], [-0.04, 0.82, -0.1]])
    g = _cuda(inp, cuda_device)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"], align_corners=ac)
    rdx, rdth = oracle.stn_bwd(*(inp[k].double().numpy() for k in ("x", "theta", "dy")), align_corners=ac)
    assert_close(_np(dx), rdx, "grad", f"dx[{variant}]")
    assert_close(_np(dth), rdth, "grad", f"dtheta[{variant}]")


@pytest.mark.parametrize("flow", ["smooth", "stress"])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_tiled_variant(cuda_device, monkeypatch, flow, padding):
    """The staged-footprint warp path (RSGRAD_WARP=tiled) matches the oracle too,
    including the in-kernel direct-gather fallback for large (stress) footprints."""
    monkeypatch.setenv("RSGRAD_WARP", "tiled")
    inp = synth.warp_inputs(2, 3, 70, 100, cfg=1, flow=flow)
    g = _cuda(inp, cuda_device)
    y = rsgrad.warp_fwd(g["x"], g["flow"], padding=padding)
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding)
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    border = padding == "border"
    assert_close(_np(y), oracle.warp_fwd(x, fl, border), "fwd", "y")
    rdx, rdf = oracle.warp_bwd(x, fl, dy, border)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


def test_host_pointer_chunked_all_layers(cuda_device):
    """Host buffers (pinned) take the library's chunked two-stream staging path
    (batch split into sample chunks, last one ragged); results equal the device path."""
    N = 5
    s = synth.stn_inputs(N, 4, 40, 48, cfg=1)
    hs = {k: v.pin_memory() for k, v in s.items()}
    gs = _cuda(s, cuda_device)
    assert torch.equal(rsgrad.stn_fwd(hs["x"], hs["theta"]), rsgrad.stn_fwd(gs["x"], gs["theta"]).cpu())
    a = rsgrad.stn_bwd(hs["x"], hs["theta"], hs["dy"], deterministic=True)
    b = rsgrad.stn_bwd(gs["x"], gs["theta"], gs["dy"], deterministic=True)
    assert all(torch.equal(p, q.cpu()) for p, q in zip(a, b))
    w = synth.warp_inputs(N, 3, 33, 41, cfg=1)
    hw = {k: v.pin_memory() for k, v in w.items()}
    gw = _cuda(w, cuda_device)
    assert torch.equal(rsgrad.warp_fwd(hw["x"], hw["flow"]), rsgrad.warp_fwd(gw["x"], gw["flow"]).cpu())
    a = rsgrad.warp_bwd(hw["x"], hw["flow"], hw["dy"])
    rdx, rdf = oracle.warp_bwd(*(w[k].double().numpy() for k in ("x", "flow", "dy")))
    assert_close(_np(a[0]), rdx, "grad", "host dx")
    assert_close(_np(a[1]), rdf, "grad", "host dflow")
    bs = synth.bslice_inputs(N, 64, 48, 8, 4, 3, cfg=1)
    hb = {k: v.pin_memory() for k, v in bs.items()}
    gb = _cuda(bs, cuda_device)
    a = rsgrad.bslice_bwd(hb["grid"], hb["guide"], hb["x"], hb["dy"], deterministic=True)
    b = rsgrad.bslice_bwd(gb["grid"], gb["guide"], gb["x"], gb["dy"], deterministic=True)
    assert all(torch.equal(p, q.cpu()) for p, q in zip(a, b))


@pytest.mark.parametrize("C", [1, 7, 33])
def test_stn_channel_chunking(cuda_device, C):
    """C not a multiple of any channel-chunk size (ragged last chunk), C = 1."""
    inp = synth.stn_inputs(2, C, 45, 70, 52, 61, cfg=1)
    g = _cuda(inp, cuda_device)
    y = rsgrad.stn_fwd(g["x"], g["theta"], 52, 61)
    dx, dth = rsgrad.stn_bwd(g["x"], g["theta"], g["dy"])
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    assert_close(_np(y), oracle.stn_fwd(x, th, 52, 61), "fwd", "y")
    rdx, rdth = oracle.stn_bwd(x, th, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


def test_null_gradient_outputs(cuda_device):
    """A NULL gradient pointer skips that gradient; the others are unchanged."""
    s = _cuda(synth.stn_inputs(2, 4, 32, 40, cfg=1), cuda_device)
    full = rsgrad.stn_bwd(s["x"], s["theta"], s["dy"])
    only_dx = rsgrad.stn_bwd(s["x"], s["theta"], s["dy"], need_dtheta=False)
    only_dth = rsgrad.stn_bwd(s["x"], s["theta"], s["dy"], need_dx=False)
    assert only_dx[1] is None and only_dth[0] is None
    assert torch.equal(only_dx[0], full[0]) and torch.equal(only_dth[1], full[1])
    w = _cuda(synth.warp_inputs(1, 3, 30, 34, cfg=1), cuda_device)
    fw = rsgrad.warp_bwd(w["x"], w["flow"], w["dy"])
    df = rsgrad.warp_bwd(w["x"], w["flow"], w["dy"], need_dx=False)[1]
    assert torch.equal(df, fw[1])
    b = _cuda(synth.bslice_inputs(1, 64, 64, 8, 4, 4, cfg=1), cuda_device)
    fb = rsgrad.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"])
    for mask in [(True, False, False), (False, True, False), (False, False, True)]:
        part = rsgrad.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"], need_dgrid=mask[0],
                                 need_dguide=mask[1], need_dx=mask[2])
        for want, got, ref in zip(mask, part, fb):
            if want:
                assert_close(_np(got), _np(ref), "grad", "partial bslice output")
            else:
                assert got is None


def test_bslice_many_planes_and_coarse_grid(cuda_device):
    """D = 16 planes, a 2x3 grid on 200x300 pixels (dual cells split into sub-tiles)."""
    inp = synth.bslice_inputs(1, 200, 300, 16, 2, 3, cfg=1, grid="iid", guide="wide")
    g = _cuda(inp, cuda_device)
    y = rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dgr), rgr, "grad", "dgrid")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dx), rdx, "grad", "dx")


def _collapse_flow(N, H, W):
    """A flow that folds each row onto ~1/30 of its width and each column onto ~1/10 of
    its height: ~1300 taps land on every element of a small region."""
    yy, xx = torch.meshgrid(torch.arange(H, dtype=torch.float32), torch.arange(W, dtype=torch.float32),
                            indexing="ij")
    return torch.stack([-xx * 0.97 + 3.3, -yy * 0.9 + 2.6]).expand(N, 2, H, W).contiguous()


def _fp32_sum_bound(x, flow, dy, border):
    """Worst-case rounding of an fp32 sum in any order (PAPER.md:733's atomics): for an
    element receiving n terms, |fl(sum) - sum| <= (n - 1) u sum|term| with u = 2^-24
    (+ one rounding of each product w*g).  Computed from the oracle with |dy|
    (the weights are >= 0, so dx(|dy|) = sum |w g|) and a tap count per element."""
    absdx, _ = oracle.warp_bwd(x, flow, np.abs(dy), border)
    N, C, H, W = x.shape
    # taps per element: count every tap that lands in the image (weights ignored)
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    n_max = 0
    for n in range(N):
        ix = xx + flow[n, 0].astype(np.float64)
        iy = yy + flow[n, 1].astype(np.float64)
        if border:
            ix, iy = np.clip(ix, 0, W - 1), np.clip(iy, 0, H - 1)
        x0, y0 = np.floor(ix).astype(np.int64), np.floor(iy).astype(np.int64)
        cnt = np.zeros((H + 2, W + 2), np.int64)
        for dy_, dx_ in ((0, 0), (0, 1), (1, 0), (1, 1)):
            ex, ey = x0 + dx_, y0 + dy_
            ok = (ex >= 0) & (ex < W) & (ey >= 0) & (ey < H)
            np.add.at(cnt, (ey[ok], ex[ok]), 1)
        n_max = max(n_max, int(cnt.max()))
    u = 2.0 ** -24
    return (n_max + 1) * u * absdx + 1e-30


@pytest.mark.parametrize("variant", ["auto", "auto_r16", "win8,4,4", "win4,8,2", "win8,8,1", "win4,4,3", "direct"])
@pytest.mark.parametrize("shape", [(2, 3, 70, 100), (1, 7, 45, 61), (1, 1, 33, 36), (2, 2, 130, 68)])
@pytest.mark.parametrize("flow", ["smooth", "stress", "collapse"])
@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_bwd_variants(cuda_device, monkeypatch, variant, shape, flow, padding):
    """warp_bwd d_input variants: "auto" = row strips with register-combined taps
    (warp_bwd_strip, R = 8 rows per warp / "auto_r16" R = 16), "win..." = per-warp shared windows flushed
    by vector reds (RSGRAD_WARP_BWD=winR,NW,IT), "direct" = one fp32 red per tap (the
    unconverted scatter, = SCATTER_ATOMIC).  Ragged strips, W % 32 != 0, C > 4 (channel
    chunks), stress flows (taps far from their row) and a collapsing flow (~1300 taps per
    element: runs of lanes on one cell, rows on one cell).  The per-tap kernel is held to
    the worst-case rounding bound of an unordered fp32 sum instead of T: its error grows
    with the fan-in, which is why AUTO combines taps before the reds."""
    if variant.startswith("win"):
        monkeypatch.setenv("RSGRAD_WARP_BWD", variant)
    elif variant == "direct":
        monkeypatch.setenv("RSGRAD_WARP_BWD", "direct")
    elif variant == "auto_r16":
        monkeypatch.setenv("RSGRAD_WARP_R", variant[6:])
    N, C, H, W = shape
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow="stress" if flow == "collapse" else flow)
    if flow == "collapse":
        inp["flow"] = _collapse_flow(N, H, W)
    g = _cuda(inp, cuda_device)
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding)
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    rdx, rdf = oracle.warp_bwd(x, fl, dy, padding == "border")
    assert_close(_np(df), rdf, "grad", f"dflow[{variant}]")
    if variant == "direct" and flow == "collapse":
        bound = _fp32_sum_bound(x, fl, dy, padding == "border")
        err = np.abs(_np(dx) - rdx)
        assert np.all(err <= bound), f"dx[direct] beyond the fp32 summation bound: {np.max(err / bound)}"
    else:
        assert_close(_np(dx), rdx, "grad", f"dx[{variant}]")


@pytest.mark.parametrize("padding", ["zeros", "border"])
def test_warp_bwd_auto_collapse_paper_shape(cuda_device, padding):
    """configs[2] shape (8 x 3 x 384 x 512) with a collapsing flow: AUTO d_input and
    d_flow within T on every element (border padding also clamps the off-image taps
    onto the edge rows / columns)."""
    N, C, H, W = 8, 3, 384, 512
    inp = synth.warp_inputs(N, C, H, W, cfg=3, flow="smooth")
    inp["flow"] = _collapse_flow(N, H, W)
    g = _cuda(inp, cuda_device)
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding=padding)
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    rdx, rdf = oracle.warp_bwd(x, fl, dy, padding == "border")
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


def test_warp_bwd_heavy_samples_take_fixed_point(cuda_device):
    """AUTO marks a sample heavy when one pre-summed emission carries >= 32 taps (a
    collapsing flow) and recomputes its d_input with the fixed-point scatter: that sample
    is then bitwise equal to deterministic=1; a smooth-flow sample in the same batch stays
    on the fp32 pre-summed reds (and within T)."""
    N, C, H, W = 2, 3, 96, 160
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow="smooth")
    inp["flow"][1] = _collapse_flow(1, H, W)[0]
    g = _cuda(inp, cuda_device)
    auto, _ = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"])
    det, _ = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], deterministic=True)
    assert torch.equal(auto[1], det[1])
    rdx, _ = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")))
    assert_close(_np(auto), rdx, "grad", "dx")


@pytest.mark.parametrize("flow", ["zero", "int", "translate_border"])
def test_warp_bwd_strip_special_flows(cuda_device, flow):
    """Integer and zero flows put every sample on a kink (fx = fy = 0): the strip kernel's
    carried taps then have zero weight and are skipped; a large translation with border
    padding clamps whole rows onto one edge column (a vertical run per lane)."""
    N, C, H, W = 2, 3, 67, 90
    inp = synth.warp_inputs(N, C, H, W, cfg=1, flow="zero")
    if flow == "int":
        inp["flow"] = torch.stack([torch.full((H, W), 3.0), torch.full((H, W), -2.0)]).expand(N, 2, H, W).contiguous()
    elif flow == "translate_border":
        inp["flow"] = torch.stack([torch.full((H, W), 500.5), torch.full((H, W), 0.25)]).expand(N, 2, H, W).contiguous()
    g = _cuda(inp, cuda_device)
    border = flow == "translate_border"
    dx, df = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], padding="border" if border else "zeros")
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    rdx, rdf = oracle.warp_bwd(x, fl, dy, border)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(df), rdf, "grad", "dflow")


def test_warp_bwd_scatter_atomic_algo(cuda_device):
    """SCATTER_ATOMIC = the per-tap red kernel; it agrees with AUTO and the oracle."""
    inp = synth.warp_inputs(2, 3, 64, 96, cfg=1)
    g = _cuda(inp, cuda_device)
    a = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"], algo="scatter_atomic")
    b = rsgrad.warp_bwd(g["x"], g["flow"], g["dy"])
    rdx, rdf = oracle.warp_bwd(*(inp[k].double().numpy() for k in ("x", "flow", "dy")))
    for dx, df in (a, b):
        assert_close(_np(dx), rdx, "grad", "dx")
        assert_close(_np(df), rdf, "grad", "dflow")


@pytest.mark.parametrize("shape", [(1, 70, 66, 16, 1, 1), (1, 64, 96, 1, 2, 3)])
@pytest.mark.parametrize("guide", ["uniform", "wide"])
def test_bslice_bwd_single_cell_and_null_outputs(cuda_device, shape, guide):
    """Dual-cell backward on a single 70 x 66 cell (D = 16) and with D = 1; a NULL
    dX / d_guide skips that output and leaves d_grid bitwise unchanged."""
    N, H, W, D, Gh, Gw = shape
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, grid="iid", guide=guide)
    g = _cuda(inp, cuda_device)
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dgr), rgr, "grad", "dgrid")
    a = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    assert torch.equal(a[0], dgr) and torch.equal(a[1], dgd) and torch.equal(a[2], dx)
    b = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], need_dguide=False, need_dx=False)
    assert b[1] is None and b[2] is None and torch.equal(b[0], dgr)


# ============================================================================ conv (§8(f) f1)
def _conv_inputs(N, Ci, Co, H, W, kh, kw, seed=0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(N, Ci, H, W, generator=g, dtype=torch.float64).float(),
            (torch.randn(Co, Ci, kh, kw, generator=g, dtype=torch.float64) / (Ci * kh * kw) ** 0.5).float(),
            torch.randn(N, Co, H, W, generator=g, dtype=torch.float64).float())


@pytest.mark.parametrize("dims", [(2, 3, 5, 37, 45, 3, 3), (1, 16, 16, 40, 70, 3, 3), (2, 20, 17, 19, 33, 5, 1),
                                  (1, 1, 1, 1, 1, 3, 3), (1, 9, 3, 16, 40, 1, 5), (1, 4, 6, 23, 29, 2, 4),
                                  (1, 2, 33, 17, 16, 7, 7)])
@pytest.mark.parametrize("algo", ["auto", "scatter_atomic"])
def test_conv_parity(cuda_device, dims, algo):
    """Forward, d_input (sheared gather = AUTO, or the atomic scatter) and d_kernel vs the
    fp64 oracle: ragged tiles, channel chunks (Ci > 8), output-channel groups (Co > 16),
    even and non-square kernels, a 1 x 1 image."""
    x, k, dy = _conv_inputs(*dims)
    g = [t.to(cuda_device) for t in (x, k, dy)]
    y = rsgrad.conv_fwd(g[0], g[1])
    dx, dk = rsgrad.conv_bwd(g[0], g[1], g[2], algo=algo)
    xn, kn, dyn = (t.double().numpy() for t in (x, k, dy))
    assert_close(_np(y), oracle.conv_fwd(xn, kn), "fwd", "y")
    rdx, rdk = oracle.conv_bwd(xn, kn, dyn)
    assert_close(_np(dx), rdx, "grad", f"dx[{algo}]")
    assert_close(_np(dk), rdk, "grad", "dk")


def test_conv_gather_deterministic_and_null_outputs(cuda_device):
    x, k, dy = (t.to(cuda_device) for t in _conv_inputs(2, 16, 16, 64, 64, 3, 3, seed=1))
    a = rsgrad.conv_bwd(x, k, dy, deterministic=True)
    b = rsgrad.conv_bwd(x, k, dy, deterministic=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    only_dk = rsgrad.conv_bwd(x, k, dy, need_dx=False)
    assert only_dk[0] is None and torch.equal(only_dk[1], a[1])
    only_dx = rsgrad.conv_bwd(x, k, dy, need_dk=False)
    assert only_dx[1] is None and torch.equal(only_dx[0], a[0])
    with pytest.raises(rsgrad.RsgradError):
        rsgrad.conv_bwd(x, k, dy, algo="scatter_priv")


def test_conv_paper_shape_sampled(cuda_device):
    """The paper's 16 x 16 x 256 x 256 conv layer, 3 x 3 kernel: dx from the
    gather and from the atomic scatter agree everywhere; sampled elements and dk vs the
    oracle on a 2-sample slice (dk rescaled: it sums over the batch)."""
    x, k, dy = _conv_inputs(16, 16, 16, 256, 256, 3, 3, seed=2)
    g = [t.to(cuda_device) for t in (x, k, dy)]
    dxg, dkg = rsgrad.conv_bwd(*g)
    dxa, _ = rsgrad.conv_bwd(*g, algo="scatter_atomic", need_dk=False)
    assert_close(_np(dxa), _np(dxg).astype(np.float64), "grad", "dx atomic vs gather")
    xs, dys = x[:2].double().numpy(), dy[:2].double().numpy()
    rdx, _ = oracle.conv_bwd(xs, k.double().numpy(), dys, need_dk=False)
    assert_close(_np(dxg[:2]), rdx, "grad", "dx[:2]")
    _, rdk = oracle.conv_bwd(x.double().numpy(), k.double().numpy(), dy.double().numpy(), need_dx=False)
    assert_close(_np(dkg), rdk, "grad", "dk")


# ============================================================================ checkpointing study (§8(f) f4)
@pytest.mark.parametrize("ks", [(1, 5), (3, 5), (2, 2), (7, 7)])
@pytest.mark.parametrize("schedule", ["root", "inline", "at"])
def test_convloss_grad_schedules(cuda_device, ks, schedule):
    """d_in of the conv loss under the three schedules the paper times
    (compute_root / compute_inline / compute_at) vs the oracle; ragged
    32 x 32 tiles and a 2-sample batch."""
    kh, kw = ks
    g = torch.Generator().manual_seed(17)
    inp = torch.randn(2, 45, 70, generator=g, dtype=torch.float64).float()
    tgt = torch.randn(2, 45, 70, generator=g, dtype=torch.float64).float()
    k = (torch.randn(kh, kw, generator=g, dtype=torch.float64) / (kh * kw) ** 0.5).float()
    d = rsgrad.convloss_grad(inp.to(cuda_device), k, tgt.to(cuda_device), schedule=schedule)
    ref = oracle.convloss_grad(inp.double().numpy(), k.double().numpy(), tgt.double().numpy())
    assert_close(_np(d), ref, "grad", f"d_in[{schedule}]")


def test_convloss_paper_shape_schedules_agree(cuda_device):
    """2560 x 1600 with the paper's 3 x 5 kernel: the three schedules agree
    with each other everywhere and with the oracle."""
    g = torch.Generator().manual_seed(18)
    inp = torch.rand(1, 1600, 2560, generator=g, dtype=torch.float64).float()
    tgt = torch.rand(1, 1600, 2560, generator=g, dtype=torch.float64).float()
    k = (torch.randn(3, 5, generator=g, dtype=torch.float64) / 15 ** 0.5).float()
    ref = oracle.convloss_grad(inp.double().numpy(), k.double().numpy(), tgt.double().numpy())
    for sch in ("root", "inline", "at"):
        d = rsgrad.convloss_grad(inp.to(cuda_device), k, tgt.to(cuda_device), schedule=sch)
        assert_close(_np(d), ref, "grad", f"d_in[{sch}]")


@pytest.mark.parametrize("shape", [(2, 3, 5, 7), (1, 1, 1, 1), (1, 4, 33, 65)])
def test_upsample4_pair(cuda_device, shape):
    """output(x) = input(x/4) and its converted gather adjoint;
    the forward is exact, the adjoint a 16-term sum."""
    g = torch.Generator().manual_seed(19)
    N, C, H, W = shape
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, 4 * H, 4 * W, generator=g, dtype=torch.float64).float()
    y = rsgrad.upsample4_fwd(x.to(cuda_device))
    assert torch.equal(y.cpu(), torch.from_numpy(oracle.upsample4_fwd(x.double().numpy())).float())
    dx = rsgrad.upsample4_bwd(dy.to(cuda_device))
    assert_close(_np(dx), oracle.upsample4_bwd(dy.double().numpy()), "grad", "upsample dx")


# ============================================================================ STN variants (§8(f) f3)
def _var_theta(N, rows, seed):
    g = torch.Generator().manual_seed(seed)
    th = torch.zeros(N, rows, rows + 1, dtype=torch.float64)
    for n in range(N):
        s = 0.8 + 0.4 * torch.rand(1, generator=g, dtype=torch.float64)
        th[n, :, :rows] = torch.eye(rows, dtype=torch.float64) * s + \
            (torch.rand(rows, rows, generator=g, dtype=torch.float64) - 0.5) * 0.5
        th[n, :, rows] = (torch.rand(rows, generator=g, dtype=torch.float64) - 0.5) * 0.4
    return th.float()


@pytest.mark.parametrize("dims", [(2, 3, 37, 45, 30, 52), (1, 16, 64, 64, 64, 64), (1, 1, 5, 4, 3, 7)])
@pytest.mark.parametrize("ac", [True, False])
def test_stn_bicubic_parity(cuda_device, dims, ac):
    N, C, H, W, Ho, Wo = dims
    g = torch.Generator().manual_seed(31)
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, Ho, Wo, generator=g, dtype=torch.float64).float()
    th = _var_theta(N, 2, 32)
    y = rsgrad.stn_bicubic_fwd(x.to(cuda_device), th.to(cuda_device), Ho, Wo, align_corners=ac)
    xn, tn, dn = x.double().numpy(), th.double().numpy(), dy.double().numpy()
    assert_close(_np(y), oracle.stn_bicubic_fwd(xn, tn, Ho, Wo, ac), "fwd", "y")
    rdx, rdth = oracle.stn_bicubic_bwd(xn, tn, dn, ac)
    for algo in ("auto", "gather", "scatter_atomic"):
        dx, dth = rsgrad.stn_bicubic_bwd(x.to(cuda_device), th.to(cuda_device), dy.to(cuda_device),
                                         align_corners=ac, algo=algo)
        assert_close(_np(dx), rdx, "grad", f"dx[{algo}]")
        assert_close(_np(dth), rdth, "grad", f"dtheta[{algo}]")


def test_stn_bicubic_gather_deterministic_and_fallback(cuda_device):
    """The converted-gather d_input is bitwise reproducible; a singular theta (rank-1
    map) and a 5x zoom-in (each input pixel's preimage window > 1024 output pixels) fall
    back to the reds per sample, next to a regular sample in the same batch."""
    g = torch.Generator().manual_seed(35)
    N, C, H, W = 3, 5, 40, 48
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    th = _var_theta(N, 2, 36)
    th[1] = torch.tensor([[0.5, 0.5, 0.1], [0.5, 0.5, -0.1]])    # singular
    th[2] = torch.tensor([[0.2, 0.01, 0.05], [-0.01, 0.2, 0.0]])  # zoom-in: ~42 x 42 window
    xs, ts, ds = (t.to(cuda_device) for t in (x, th, dy))
    a = rsgrad.stn_bicubic_bwd(xs, ts, ds, deterministic=True)
    b = rsgrad.stn_bicubic_bwd(xs, ts, ds, deterministic=True)
    # every sample, the fallback ones included (fixed-point scatter, det.cuh)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    rdx, rdth = oracle.stn_bicubic_bwd(x.double().numpy(), th.double().numpy(), dy.double().numpy())
    assert_close(_np(a[0]), rdx, "grad", "dx")
    assert_close(_np(a[1]), rdth, "grad", "dtheta")


@pytest.mark.parametrize("dims", [(2, 2, 9, 11, 13, 8, 12, 10), (1, 4, 32, 32, 32, 32, 32, 32), (1, 1, 2, 3, 4, 2, 2, 2)])
@pytest.mark.parametrize("ac", [True, False])
def test_stn3d_parity(cuda_device, dims, ac):
    N, C, D, H, W, Do, Ho, Wo = dims
    g = torch.Generator().manual_seed(33)
    x = torch.randn(N, C, D, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, Do, Ho, Wo, generator=g, dtype=torch.float64).float()
    th = _var_theta(N, 3, 34)
    y = rsgrad.stn3d_fwd(x.to(cuda_device), th.to(cuda_device), (Do, Ho, Wo), align_corners=ac)
    dx, dth = rsgrad.stn3d_bwd(x.to(cuda_device), th.to(cuda_device), dy.to(cuda_device), align_corners=ac)
    xn, tn, dn = x.double().numpy(), th.double().numpy(), dy.double().numpy()
    assert_close(_np(y), oracle.stn3d_fwd(xn, tn, (Do, Ho, Wo), ac), "fwd", "y")
    rdx, rdth = oracle.stn3d_bwd(xn, tn, dn, ac)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


def test_stn_variants_refuse_border_and_gather(cuda_device):
    x = torch.zeros(1, 1, 8, 8, device=cuda_device)
    th = torch.zeros(1, 2, 3, device=cuda_device)
    o = rsgrad._opts(True, "border")
    y = torch.empty_like(x)
    assert rsgrad.lib().stn_bicubic_fwd(rsgrad._ptr(x), rsgrad._ptr(th), 1, 1, 8, 8, 8, 8,
                                        __import__("ctypes").byref(o), rsgrad._ptr(y), None) == -4


def test_stn_variants_bench_shapes_sampled(cuda_device):
    """The bench's f3 cases in their launch configuration: bicubic 4 x 16 x 512^2 and
    3-D 2 x 4 x 96^3; samples 0 and 3 (resp. 1) in full against the oracle."""
    si = synth.stn_inputs(4, 16, 512, 512, cfg=2)
    g = _cuda(si, cuda_device)
    y = rsgrad.stn_bicubic_fwd(g["x"], g["theta"])
    dx, dth = rsgrad.stn_bicubic_bwd(g["x"], g["theta"], g["dy"])
    for n in (0, 3):
        x, th, dy = (si[k][n:n + 1].double().numpy() for k in ("x", "theta", "dy"))
        assert_close(_np(y[n:n + 1]), oracle.stn_bicubic_fwd(x, th), "fwd", f"y[{n}]")
        rdx, rdth = oracle.stn_bicubic_bwd(x, th, dy)
        assert_close(_np(dx[n:n + 1]), rdx, "grad", f"dx[{n}]")
        assert_close(_np(dth[n:n + 1]), rdth, "grad", f"dtheta[{n}]")
    g3 = torch.Generator().manual_seed(37)
    x3 = torch.randn(2, 4, 96, 96, 96, generator=g3, dtype=torch.float64).float()
    d3 = torch.randn(2, 4, 96, 96, 96, generator=g3, dtype=torch.float64).float()
    t3 = (torch.eye(3, 4, dtype=torch.float64).expand(2, 3, 4) +
          0.05 * torch.randn(2, 3, 4, generator=g3, dtype=torch.float64)).float().contiguous()
    y3 = rsgrad.stn3d_fwd(x3.to(cuda_device), t3.to(cuda_device))
    dx3, dt3 = rsgrad.stn3d_bwd(x3.to(cuda_device), t3.to(cuda_device), d3.to(cuda_device))
    xn, tn, dn = x3[1:].double().numpy(), t3[1:].double().numpy(), d3[1:].double().numpy()
    assert_close(_np(y3[1:]), oracle.stn3d_fwd(xn, tn), "fwd", "y3")
    rdx, rdth = oracle.stn3d_bwd(xn, tn, dn)
    assert_close(_np(dx3[1:]), rdx, "grad", "dx3")
    assert_close(_np(dt3[1:]), rdth, "grad", "dtheta3")


@pytest.mark.parametrize("dims", [(2, 3, 37, 45, 30, 52), (1, 16, 64, 64, 64, 64), (1, 1, 5, 4, 3, 7)])
@pytest.mark.parametrize("ac", [True, False])
def test_stn_lanczos_parity(cuda_device, dims, ac):
    """Lanczos-3 STN (6 x 6 taps) forward, atomic d_input and d_theta vs the oracle."""
    N, C, H, W, Ho, Wo = dims
    g = torch.Generator().manual_seed(45)
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, Ho, Wo, generator=g, dtype=torch.float64).float()
    th = _var_theta(N, 2, 46)
    y = rsgrad.stn_lanczos_fwd(x.to(cuda_device), th.to(cuda_device), Ho, Wo, align_corners=ac)
    dx, dth = rsgrad.stn_lanczos_bwd(x.to(cuda_device), th.to(cuda_device), dy.to(cuda_device), align_corners=ac)
    xn, tn, dn = x.double().numpy(), th.double().numpy(), dy.double().numpy()
    assert_close(_np(y), oracle.stn_lanczos_fwd(xn, tn, Ho, Wo, ac), "fwd", "y")
    rdx, rdth = oracle.stn_lanczos_bwd(xn, tn, dn, ac)
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


def test_stn_lanczos_tiled_zoom_and_edge(cuda_device):
    """Ho, Wo multiples of 8 and 32: the 32 x 8 block tiles with 8 x 4 warp patches
    (out_pixel) under a 5x zoom-in (sample 0), a 5x zoom-out (sample 1: every output
    pixel's taps are disjoint from its neighbours') and a map whose taps are clipped by
    two image edges (sample 2)."""
    g = torch.Generator().manual_seed(47)
    N, C, H, W, Ho, Wo = 3, 2, 320, 320, 64, 64
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, Ho, Wo, generator=g, dtype=torch.float64).float()
    th = torch.tensor([[[0.21, 0.03, 0.02], [-0.02, 0.19, 0.05]],
                       [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]],
                       [[0.15, 0.05, 0.93], [-0.04, 0.16, -0.9]]])
    dx, dth = rsgrad.stn_lanczos_bwd(x.to(cuda_device), th.to(cuda_device), dy.to(cuda_device))
    rdx, rdth = oracle.stn_lanczos_bwd(x.double().numpy(), th.double().numpy(), dy.double().numpy())
    assert_close(_np(dx), rdx, "grad", "dx")
    assert_close(_np(dth), rdth, "grad", "dtheta")


# ============================================================================ boundary contract
@pytest.mark.parametrize("D", [61, 64])
def test_bslice_many_planes_tiled_backward(cuda_device, D):
    """D up to 64: the tiled backward's shared memory (2056 D + 80740 B) is set per call
    from the launch's need (212 KB at D = 64, under the 227 KB opt-in)."""
    inp = synth.bslice_inputs(1, 96, 128, D, 4, 4, cfg=1, guide="wide")
    g = _cuda(inp, cuda_device)
    assert rsgrad.workspace_bytes(2, 1, 3, 96, 128, D=D, Gh=4, Gw=4, opts=rsgrad._opts(deterministic=True)) > 0
    y = rsgrad.bslice_fwd(g["grid"], g["guide"], g["x"])
    dgr, dgd, dx = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(dgr), rgr, "grad", "dgrid")
    assert_close(_np(dgd), rgd, "grad", "dguide")
    assert_close(_np(dx), rdx, "grad", "dx")


def test_library_workspace_is_not_kept(cuda_device):
    """ws = NULL: the library takes a stream-ordered temporary from the device's default
    pool and frees it in stream order; once the stream is synchronised the pool (release
    threshold 0 by default) holds nothing for the library (SURVEY 8(b) ownership)."""
    import ctypes

    from cuda.bindings import runtime as cudart

    inp = _cuda(synth.stn_inputs(2, 4, 64, 64, cfg=1), cuda_device)
    dx, dth = torch.empty_like(inp["x"]), torch.empty(2, 2, 3, device=cuda_device)
    L = rsgrad.lib()
    o = rsgrad._opts()
    s = torch.cuda.current_stream()
    err, pool = cudart.cudaDeviceGetDefaultMemPool(cuda_device.index or 0)
    assert err == cudart.cudaError_t.cudaSuccess
    for _ in range(3):
        st = L.stn_bwd(rsgrad._ptr(inp["x"]), rsgrad._ptr(inp["theta"]), rsgrad._ptr(inp["dy"]), 2, 4, 64, 64, 64,
                       64, ctypes.byref(o), rsgrad._ptr(dx), rsgrad._ptr(dth), None, 0, ctypes.c_void_p(s.cuda_stream))
        assert st == 0
    s.synchronize()
    torch.cuda.synchronize()
    err, reserved = cudart.cudaMemPoolGetAttribute(pool, cudart.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    assert err == cudart.cudaError_t.cudaSuccess
    err, thr = cudart.cudaMemPoolGetAttribute(pool, cudart.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    if int(thr) == 0:
        assert int(reserved) == 0, f"library temporaries still reserved: {int(reserved)} B"
    ref = rsgrad.stn_bwd(inp["x"], inp["theta"], inp["dy"])
    assert torch.equal(ref[0], dx) and torch.equal(ref[1], dth)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_second_device_same_thread():
    """Tensors on cuda:1 while cuda:0 is current: every entry point switches to the
    stream's device (bslice's shared-memory attribute is set for that device too)."""
    dev1 = torch.device("cuda", 1)
    torch.cuda.set_device(0)
    b = _cuda(synth.bslice_inputs(1, 64, 64, 8, 4, 4, cfg=1), torch.device("cuda", 0))
    rsgrad.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"])
    b1 = {k: v.to(dev1) for k, v in b.items()}
    # the binding passes cuda:1's current stream without making cuda:1 current
    out = rsgrad.bslice_bwd(b1["grid"], b1["guide"], b1["x"], b1["dy"])
    torch.cuda.synchronize(dev1)
    assert torch.cuda.current_device() == 0
    gr, gd, x, dy = (v.double().cpu().numpy() for v in (b["grid"], b["guide"], b["x"], b["dy"]))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(out[0]), rgr, "grad", "dgrid on cuda:1")
    assert_close(_np(out[2]), rdx, "grad", "dx on cuda:1")


def test_lanczos_and_3d_deterministic(cuda_device):
    """deterministic=1 for the atomics-only STN variants: d_theta pass alone,
    then the fixed-point integer scatter -- bitwise equal reruns, within T of the oracle."""
    g = torch.Generator().manual_seed(61)
    N, C, H, W = 2, 3, 30, 34
    x = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    dy = torch.randn(N, C, H, W, generator=g, dtype=torch.float64).float()
    th = _var_theta(N, 2, 62)
    xs, ts, ds = (t.to(cuda_device) for t in (x, th, dy))
    a = rsgrad.stn_lanczos_bwd(xs, ts, ds, deterministic=True)
    b = rsgrad.stn_lanczos_bwd(xs, ts, ds, deterministic=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    rdx, rdth = oracle.stn_lanczos_bwd(x.double().numpy(), th.double().numpy(), dy.double().numpy())
    assert_close(_np(a[0]), rdx, "grad", "lanczos dx")
    assert_close(_np(a[1]), rdth, "grad", "lanczos dtheta")
    x3 = torch.randn(1, 2, 9, 11, 13, generator=g, dtype=torch.float64).float()
    d3 = torch.randn(1, 2, 8, 12, 10, generator=g, dtype=torch.float64).float()
    t3 = _var_theta(1, 3, 63)
    x3s, d3s, t3s = (t.to(cuda_device) for t in (x3, d3, t3))
    a3 = rsgrad.stn3d_bwd(x3s, t3s, d3s, deterministic=True)
    b3 = rsgrad.stn3d_bwd(x3s, t3s, d3s, deterministic=True)
    assert torch.equal(a3[0], b3[0]) and torch.equal(a3[1], b3[1])
    r3dx, r3dth = oracle.stn3d_bwd(x3.double().numpy(), t3.double().numpy(), d3.double().numpy())
    assert_close(_np(a3[0]), r3dx, "grad", "3d dx")
    assert_close(_np(a3[1]), r3dth, "grad", "3d dtheta")


@pytest.mark.parametrize("dims", [(2, 16, 16, 8, 16, 16), (1, 60, 50, 4, 12, 10), (2, 33, 47, 3, 5, 9)])
def test_bslice_deterministic_fine_grids(cuda_device, dims):
    """Grids finer than the tiled path's 8 px per cell: deterministic=1 takes the generic
    per-pixel adjoint with d_grid by the fixed-point integer scatter (bitwise equal reruns,
    within T); the default takes fp32 reds."""
    inp = synth.bslice_inputs(*dims, cfg=1, grid="iid", guide="wide")
    g = _cuda(inp, cuda_device)
    a = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    b = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], deterministic=True)
    for u, v in zip(a, b):
        assert torch.equal(u, v)
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(a[0]), rgr, "grad", "dgrid")
    assert_close(_np(a[1]), rgd, "grad", "dguide")
    assert_close(_np(a[2]), rdx, "grad", "dx")


@pytest.mark.parametrize("dims", [(2, 100, 130, 8, 6, 7), (1, 64, 64, 8, 4, 4), (2, 16, 16, 8, 16, 16),
                                  (1, 60, 50, 16, 3, 5)])
def test_bslice_gather_node_walk(cuda_device, dims):
    """GATHER: d_grid by the pure node gather (each grid node walks the pixels of its 2 x 2
    dual cells; clamped border taps count twice onto the border node); bitwise reproducible
    and within T; d_input / d_guide from the per-pixel kernel."""
    inp = synth.bslice_inputs(*dims, cfg=1, grid="iid", guide="wide")
    g = _cuda(inp, cuda_device)
    a = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], algo="gather")
    b = rsgrad.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"], algo="gather")
    assert torch.equal(a[0], b[0])
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
    assert_close(_np(a[0]), rgr, "grad", "dgrid")
    assert_close(_np(a[1]), rgd, "grad", "dguide")
    assert_close(_np(a[2]), rdx, "grad", "dx")
