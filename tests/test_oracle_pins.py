"""Pins for the fp64 oracle (oracle/oracle.c) against things other than itself.

Each group below anchors the oracle to what the paper and the mathematics fix:
  * hand-worked golden fixtures (tests/golden/*.json, each citing PAPER.md);
  * special cases that reduce to an independent library routine (torch fp64
    affine_grid / grid_sample / autograd — the routines the paper benchmarks
    the STN against);
  * closed forms (identity theta, quarter-pixel shift, zero / integer flow,
    constant grid);
  * the adjoint identity <A x, y> = <x, A^T y> and a brute-force operator
    matrix (reverse mode = transpose);
  * central finite differences (Eq. finite_difference);
  * invariants (partition of unity of the tent weights; warp with the
    theta-induced flow equals the STN).
A plausible mistake anywhere in the oracle (dropped tap, swapped fx/fy, wrong
unnormalisation scale, wrong clamp, transposed coefficient index) fails at least
one of them.  No GPU needed.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _np(t):
    return t.detach().double().numpy()


# --------------------------------------------------------------------------- golden
def test_golden_stn():
    g = _load("stn_halfpx_2x2.json")
    y = oracle.stn_fwd(g["x"], g["theta"], align_corners=bool(g["align_corners"]))
    np.testing.assert_array_equal(y, np.array(g["y"]))
    dx, dth = oracle.stn_bwd(g["x"], g["theta"], g["dy"], align_corners=True)
    np.testing.assert_array_equal(dx, np.array(g["dx"]))
    np.testing.assert_array_equal(dth, np.array(g["dtheta"]))


def test_golden_warp():
    g = _load("warp_2x3.json")
    y = oracle.warp_fwd(g["x"], g["flow"])
    np.testing.assert_array_equal(y, np.array(g["y"]))
    dx, df = oracle.warp_bwd(g["x"], g["flow"], g["dy"])
    np.testing.assert_array_equal(dx, np.array(g["dx"]))
    np.testing.assert_array_equal(df, np.array(g["dflow"]))


def test_golden_bslice():
    g = _load("bslice_1x2.json")
    y = oracle.bslice_fwd(g["grid"], g["guide"], g["x"])
    np.testing.assert_allclose(y, np.array(g["y"]), rtol=0, atol=1e-15)
    dgr, dgd, dx = oracle.bslice_bwd(g["grid"], g["guide"], g["x"], g["dy"])
    np.testing.assert_allclose(dx, np.array(g["dx"]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(dgd, np.array(g["dguide"]), rtol=0, atol=1e-13)
    np.testing.assert_allclose(dgr, np.array(g["dgrid"]), rtol=0, atol=1e-15)


# --------------------------------------------------------------------------- torch library pins
def _torch_stn(x, theta, dy, Ho, Wo, ac, border):
    x = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    th = torch.tensor(theta, dtype=torch.float64, requires_grad=True)
    N, C = x.shape[:2]
    grid = F.affine_grid(th, (N, C, Ho, Wo), align_corners=ac)
    y = F.grid_sample(x, grid, mode="bilinear", padding_mode="border" if border else "zeros",
                      align_corners=ac)
    y.backward(torch.tensor(dy, dtype=torch.float64))
    return _np(y), _np(x.grad), _np(th.grad)


@pytest.mark.parametrize("ac", [True, False])
@pytest.mark.parametrize("border", [False, True])
@pytest.mark.parametrize("shape", [(2, 3, 16, 16, 16, 16), (1, 2, 9, 13, 11, 7)])
def test_stn_vs_torch(ac, border, shape):
    N, C, H, W, Ho, Wo = shape
    inp = synth.stn_inputs(N, C, H, W, Ho, Wo, cfg=1)
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    ry, rdx, rdth = _torch_stn(x, th, dy, Ho, Wo, ac, border)
    y = oracle.stn_fwd(x, th, Ho, Wo, align_corners=ac, border=border)
    dx, dth = oracle.stn_bwd(x, th, dy, align_corners=ac, border=border)
    np.testing.assert_allclose(y, ry, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dx, rdx, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dth, rdth, rtol=1e-10, atol=1e-10)


def _torch_warp(x, flow, dy, border):
    x = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    fl = torch.tensor(flow, dtype=torch.float64, requires_grad=True)
    N, C, H, W = x.shape
    xs = torch.arange(W, dtype=torch.float64).view(1, 1, W)
    ys = torch.arange(H, dtype=torch.float64).view(1, H, 1)
    gx = 2.0 * (xs + fl[:, 0]) / (W - 1) - 1.0
    gy = 2.0 * (ys + fl[:, 1]) / (H - 1) - 1.0
    grid = torch.stack([gx, gy], dim=-1)
    y = F.grid_sample(x, grid, mode="bilinear", padding_mode="border" if border else "zeros",
                      align_corners=True)
    y.backward(torch.tensor(dy, dtype=torch.float64))
    return _np(y), _np(x.grad), _np(fl.grad)


@pytest.mark.parametrize("border", [False, True])
@pytest.mark.parametrize("flow", ["smooth", "stress"])
def test_warp_vs_torch(border, flow):
    inp = synth.warp_inputs(2, 3, 24, 40, cfg=1, flow=flow)
    x, fl, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    ry, rdx, rdf = _torch_warp(x, fl, dy, border)
    y = oracle.warp_fwd(x, fl, border=border)
    dx, df = oracle.warp_bwd(x, fl, dy, border=border)
    np.testing.assert_allclose(y, ry, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dx, rdx, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(df, rdf, rtol=1e-10, atol=1e-10)


def _torch_bslice(grid, guide, x, dy):
    gr = torch.tensor(grid, dtype=torch.float64, requires_grad=True)
    gd = torch.tensor(guide, dtype=torch.float64, requires_grad=True)
    xx = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    N, _, H, W = xx.shape
    xs = (2.0 * (torch.arange(W, dtype=torch.float64) + 0.5) / W - 1.0).view(1, 1, W).expand(N, H, W)
    ys = (2.0 * (torch.arange(H, dtype=torch.float64) + 0.5) / H - 1.0).view(1, H, 1).expand(N, H, W)
    gz = 2.0 * gd - 1.0
    samp = torch.stack([xs, ys, gz], dim=-1).unsqueeze(1)  # N x 1 x H x W x 3 (x, y, z)
    A = F.grid_sample(gr, samp, mode="bilinear", padding_mode="border", align_corners=False)
    A = A[:, :, 0].reshape(N, 3, 4, H, W)
    xt = torch.cat([xx, torch.ones_like(xx[:, :1])], dim=1)
    y = torch.einsum("noihw,nihw->nohw", A, xt)
    y.backward(torch.tensor(dy, dtype=torch.float64))
    return _np(y), _np(gr.grad), _np(gd.grad), _np(xx.grad)


@pytest.mark.parametrize("dims", [(2, 32, 48, 8, 4, 6), (1, 17, 23, 3, 5, 2), (1, 8, 8, 4, 16, 16)])
@pytest.mark.parametrize("guide", ["uniform", "wide"])
def test_bslice_vs_torch(dims, guide):
    N, H, W, D, Gh, Gw = dims
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, grid="iid", guide=guide)
    gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    ry, rdgr, rdgd, rdx = _torch_bslice(gr, gd, x, dy)
    y = oracle.bslice_fwd(gr, gd, x)
    dgr, dgd, dx = oracle.bslice_bwd(gr, gd, x, dy)
    np.testing.assert_allclose(y, ry, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dx, rdx, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dgr, rdgr, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(dgd, rdgd, rtol=1e-10, atol=1e-10)


# --------------------------------------------------------------------------- closed forms
def test_stn_identity_theta():
    """Identity theta: Y = X and dX = G (not bitwise: normalisation round-trips)."""
    inp = synth.stn_inputs(2, 3, 16, 20, cfg=1, theta_kind="identity")
    x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    np.testing.assert_allclose(oracle.stn_fwd(x, th), x, rtol=0, atol=1e-13)
    dx, _ = oracle.stn_bwd(x, th, dy)
    np.testing.assert_allclose(dx, dy, rtol=0, atol=1e-13)


def test_stn_quarter_pixel_closed_form():
    """theta = [[1,0,.5/(W-1)],[0,1,.5/(H-1)]] (ac=1) shifts by a quarter pixel:
    Y = 9/16 X + 3/16 X(x+1) + 3/16 X(y+1) + 1/16 X(y+1,x+1) with zero fill;
    dtheta from forward differences of X (SURVEY.md 8(c) Pins, F5)."""
    N, C, H, W = 1, 2, 12, 10
    rng = np.random.default_rng(5)
    x = rng.standard_normal((N, C, H, W))
    g = rng.standard_normal((N, C, H, W))
    th = np.array([[[1.0, 0.0, 0.5 / (W - 1)], [0.0, 1.0, 0.5 / (H - 1)]]])
    xp = np.zeros((N, C, H + 1, W + 1))
    xp[:, :, :H, :W] = x
    R, D_, B = xp[:, :, :H, 1:W + 1], xp[:, :, 1:H + 1, :W], xp[:, :, 1:H + 1, 1:W + 1]
    yref = 9 / 16 * x + 3 / 16 * R + 3 / 16 * D_ + 1 / 16 * B
    np.testing.assert_allclose(oracle.stn_fwd(x, th), yref, rtol=0, atol=1e-13)
    dix = (g * (0.75 * (R - x) + 0.25 * (B - D_))).sum(1)[0]
    diy = (g * (0.75 * (D_ - x) + 0.25 * (B - R))).sum(1)[0]
    dgx, dgy = dix * (W - 1) / 2, diy * (H - 1) / 2
    xt = np.linspace(-1, 1, W)[None, :].repeat(H, 0)
    yt = np.linspace(-1, 1, H)[:, None].repeat(W, 1)
    ref = np.array([[(dgx * xt).sum(), (dgx * yt).sum(), dgx.sum()],
                    [(dgy * xt).sum(), (dgy * yt).sum(), dgy.sum()]])
    _, dth = oracle.stn_bwd(x, th, g)
    np.testing.assert_allclose(dth[0], ref, rtol=1e-12, atol=1e-11)


def test_warp_zero_and_integer_flow():
    inp = synth.warp_inputs(2, 3, 9, 11, cfg=1, flow="zero")
    x, fl, g = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
    np.testing.assert_array_equal(oracle.warp_fwd(x, fl), x)
    dx, df = oracle.warp_bwd(x, fl, g)
    np.testing.assert_array_equal(dx, g)
    xr = np.concatenate([x[..., 1:], np.zeros_like(x[..., :1])], -1)   # X(x+1), zero at W
    xd = np.concatenate([x[:, :, 1:], np.zeros_like(x[:, :, :1])], -2)  # X(y+1), zero at H
    np.testing.assert_allclose(df[:, 0], (g * (xr - x)).sum(1), rtol=0, atol=1e-14)
    np.testing.assert_allclose(df[:, 1], (g * (xd - x)).sum(1), rtol=0, atol=1e-14)
    # integer flow (+1, -2): exact shift with zero fill
    fl2 = np.zeros_like(fl)
    fl2[:, 0], fl2[:, 1] = 1.0, -2.0
    ref = np.zeros_like(x)
    ref[:, :, 2:, :-1] = x[:, :, :-2, 1:]
    np.testing.assert_array_equal(oracle.warp_fwd(x, fl2), ref)


def test_bslice_constant_grid():
    """Constant grid A: Y = A [X;1], dX = A^T G, dguide = 0."""
    N, H, W, D, Gh, Gw = 2, 13, 17, 4, 3, 5
    inp = synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, guide="wide")
    gd, x, g = (inp[k].double().numpy() for k in ("guide", "x", "dy"))
    A = np.random.default_rng(1).standard_normal((N, 3, 4))
    grid = np.broadcast_to(A.reshape(N, 12, 1, 1, 1), (N, 12, D, Gh, Gw)).copy()
    xt = np.concatenate([x, np.ones_like(x[:, :1])], 1)
    yref = np.einsum("noi,nihw->nohw", A, xt)
    np.testing.assert_allclose(oracle.bslice_fwd(grid, gd, x), yref, rtol=0, atol=1e-13)
    _, dgd, dx = oracle.bslice_bwd(grid, gd, x, g)
    np.testing.assert_allclose(dx, np.einsum("noi,nohw->nihw", A[:, :, :3], g), rtol=0, atol=1e-13)
    np.testing.assert_allclose(dgd, 0.0, rtol=0, atol=1e-13)


# --------------------------------------------------------------------------- invariants
def test_bslice_dgrid_partition_of_unity():
    """sum over cells of dgrid = sum over pixels of G (x) [X;1], any grid."""
    inp = synth.bslice_inputs(2, 20, 28, 6, 4, 5, cfg=1, grid="iid", guide="wide")
    gr, gd, x, g = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    dgr, _, _ = oracle.bslice_bwd(gr, gd, x, g, need_dguide=False, need_dx=False)
    xt = np.concatenate([x, np.ones_like(x[:, :1])], 1)
    ref = np.einsum("nohw,nihw->noi", g, xt).reshape(2, 12)
    np.testing.assert_allclose(dgr.sum(axis=(2, 3, 4)), ref, rtol=1e-12, atol=1e-11)


def test_warp_with_theta_flow_equals_stn():
    N, C, H, W = 2, 3, 14, 18
    inp = synth.stn_inputs(N, C, H, W, cfg=1)
    x, th, g = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
    jj, ii = np.meshgrid(np.arange(W), np.arange(H))
    xt, yt = -1 + 2 * jj / (W - 1), -1 + 2 * ii / (H - 1)
    flow = np.empty((N, 2, H, W))
    for n in range(N):
        gx = th[n, 0, 0] * xt + th[n, 0, 1] * yt + th[n, 0, 2]
        gy = th[n, 1, 0] * xt + th[n, 1, 1] * yt + th[n, 1, 2]
        flow[n, 0] = (gx + 1) * (W - 1) / 2 - jj
        flow[n, 1] = (gy + 1) * (H - 1) / 2 - ii
    np.testing.assert_allclose(oracle.warp_fwd(x, flow), oracle.stn_fwd(x, th), rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.warp_bwd(x, flow, g)[0], oracle.stn_bwd(x, th, g)[0],
                               rtol=0, atol=1e-12)


def test_adjoint_identity_all_layers():
    """<A x, y> = <x, A^T y>: each layer is linear in X (and bslice in grid)."""
    i = synth.stn_inputs(2, 3, 15, 17, 13, 19, cfg=1)
    x, th, g = (i[k].double().numpy() for k in ("x", "theta", "dy"))
    for ac in (True, False):
        for border in (False, True):
            lhs = np.vdot(oracle.stn_fwd(x, th, 13, 19, ac, border), g)
            rhs = np.vdot(x, oracle.stn_bwd(x, th, g, ac, border)[0])
            assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)
    i = synth.warp_inputs(2, 3, 15, 17, cfg=1, flow="stress")
    x, fl, g = (i[k].double().numpy() for k in ("x", "flow", "dy"))
    lhs, rhs = np.vdot(oracle.warp_fwd(x, fl), g), np.vdot(x, oracle.warp_bwd(x, fl, g)[0])
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)
    i = synth.bslice_inputs(2, 15, 17, 4, 3, 5, cfg=1, grid="iid")
    gr, gd, x, g = (i[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    zero = np.zeros_like(x)
    # linear in X after removing the bias (X=0) response
    lhs = np.vdot(oracle.bslice_fwd(gr, gd, x) - oracle.bslice_fwd(gr, gd, zero), g)
    rhs = np.vdot(x, oracle.bslice_bwd(gr, gd, x, g)[2])
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)
    # linear in the grid
    lhs = np.vdot(oracle.bslice_fwd(gr, gd, x), g)
    rhs = np.vdot(gr, oracle.bslice_bwd(gr, gd, x, g)[0])
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


def test_stn_brute_force_operator_matrix():
    """Materialise M from forward calls on basis vectors; dX must equal M^T G."""
    N, C, H, W, Ho, Wo = 1, 2, 6, 7, 5, 8
    i = synth.stn_inputs(N, C, H, W, Ho, Wo, cfg=1)
    th, g = i["theta"].double().numpy(), i["dy"].double().numpy()
    for ac in (True, False):
        cols = []
        for k in range(C * H * W):
            e = np.zeros(C * H * W)
            e[k] = 1.0
            cols.append(oracle.stn_fwd(e.reshape(N, C, H, W), th, Ho, Wo, ac).ravel())
        M = np.stack(cols, 1)
        dx, _ = oracle.stn_bwd(np.zeros((N, C, H, W)), th, g, ac)
        np.testing.assert_allclose(dx.ravel(), M.T @ g.ravel(), rtol=0, atol=1e-13)


# --------------------------------------------------------------------------- central FD
def _min_kink_dist(v):
    return float(np.min(np.abs(v - np.round(v))))


def test_stn_theta_central_fd():
    N, C, H, W = 1, 3, 16, 16   # configs[0]: STN 1x3x16x16
    i = synth.stn_inputs(N, C, H, W, cfg=1)
    x, th, g = (i[k].double().numpy() for k in ("x", "theta", "dy"))
    for ac in (True, False):
        # sample coordinates must stay >= 1e-3 px from kinks for FD to be valid
        jj, ii = np.meshgrid(np.arange(W), np.arange(H))
        xt = -1 + 2 * jj / (W - 1) if ac else (2 * jj + 1) / W - 1
        yt = -1 + 2 * ii / (H - 1) if ac else (2 * ii + 1) / H - 1
        t = th[0]
        s = (W - 1) / 2 if ac else W / 2
        ix = (t[0, 0] * xt + t[0, 1] * yt + t[0, 2] + 1) * s - (0 if ac else 0.5)
        assert _min_kink_dist(ix) > 1e-4
        _, dth = oracle.stn_bwd(x, th, g, ac)
        h = 1e-6
        fd = np.zeros_like(th)
        for k in range(6):
            tp, tm = th.copy(), th.copy()
            tp.reshape(-1)[k] += h
            tm.reshape(-1)[k] -= h
            fd.reshape(-1)[k] = (np.vdot(oracle.stn_fwd(x, tp, align_corners=ac), g) -
                                 np.vdot(oracle.stn_fwd(x, tm, align_corners=ac), g)) / (2 * h)
        np.testing.assert_allclose(dth, fd, rtol=1e-6, atol=1e-6)


def test_warp_flow_central_fd():
    i = synth.warp_inputs(1, 3, 8, 9, cfg=1, flow="stress")
    x, fl, g = (i[k].double().numpy() for k in ("x", "flow", "dy"))
    assert _min_kink_dist(fl) > 1e-4
    _, df = oracle.warp_bwd(x, fl, g)
    h = 1e-6
    fd = np.zeros_like(fl)
    for k in range(fl.size):
        fp, fm = fl.copy(), fl.copy()
        fp.reshape(-1)[k] += h
        fm.reshape(-1)[k] -= h
        fd.reshape(-1)[k] = (np.vdot(oracle.warp_fwd(x, fp), g) - np.vdot(oracle.warp_fwd(x, fm), g)) / (2 * h)
    np.testing.assert_allclose(df, fd, rtol=1e-6, atol=1e-7)


def test_bslice_guide_central_fd():
    i = synth.bslice_inputs(1, 6, 7, 4, 3, 2, cfg=1, grid="iid", guide="wide")
    gr, gd, x, g = (i[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
    assert _min_kink_dist(gd * 4 - 0.5) > 1e-4
    _, dgd, _ = oracle.bslice_bwd(gr, gd, x, g)
    h = 1e-6
    fd = np.zeros_like(gd)
    for k in range(gd.size):
        p, m = gd.copy(), gd.copy()
        p.reshape(-1)[k] += h
        m.reshape(-1)[k] -= h
        fd.reshape(-1)[k] = (np.vdot(oracle.bslice_fwd(gr, p, x), g) -
                             np.vdot(oracle.bslice_fwd(gr, m, x), g)) / (2 * h)
    np.testing.assert_allclose(dgd, fd, rtol=1e-6, atol=1e-7)


def test_fd_negative_control_at_kink():
    """At an exact kink (zero flow) central FD returns the central difference,
    which differs from the floor-cell (right) derivative the oracle pins (P2)."""
    x = np.zeros((1, 1, 1, 3))
    x[0, 0, 0] = [0.0, 1.0, 5.0]
    fl = np.zeros((1, 2, 1, 3))
    g = np.zeros((1, 1, 1, 3))
    g[0, 0, 0, 1] = 1.0
    _, df = oracle.warp_bwd(x, fl, g)
    assert df[0, 0, 0, 1] == 4.0          # right derivative X(2)-X(1)
    h = 1e-6
    fp, fm = fl.copy(), fl.copy()
    fp[0, 0, 0, 1] += h
    fm[0, 0, 0, 1] -= h
    fd = (np.vdot(oracle.warp_fwd(x, fp), g) - np.vdot(oracle.warp_fwd(x, fm), g)) / (2 * h)
    assert abs(fd - 2.5) < 1e-6            # central: (4 + 1)/2


# --------------------------------------------------------------------------- conv layer (§8(f) f1)
def _conv_case(N, Ci, Co, H, W, kh, kw, seed=0):
    g = np.random.default_rng(seed)
    return (g.standard_normal((N, Ci, H, W)), g.standard_normal((Co, Ci, kh, kw)),
            g.standard_normal((N, Co, H, W)))


@pytest.mark.parametrize("dims", [(2, 3, 4, 9, 11, 3, 3), (1, 2, 2, 12, 10, 1, 5), (1, 1, 3, 8, 8, 3, 5),
                                  (2, 4, 1, 6, 7, 5, 1)])
def test_conv_vs_torch(dims):
    """Odd kernels: the layer is torch's conv2d (a cross-correlation) with the kernel
    flipped in both axes and padding k//2; dx and dk from torch autograd (fp64)."""
    N, Ci, Co, H, W, kh, kw = dims
    x, k, dy = _conv_case(*dims)
    xt = torch.tensor(x, requires_grad=True)
    kt = torch.tensor(k, requires_grad=True)
    yt = F.conv2d(xt, kt.flip(-1, -2), padding=(kh // 2, kw // 2))
    yt.backward(torch.tensor(dy))
    np.testing.assert_allclose(oracle.conv_fwd(x, k), _np(yt), rtol=1e-12, atol=1e-12)
    dx, dk = oracle.conv_bwd(x, k, dy)
    np.testing.assert_allclose(dx, _np(xt.grad), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dk, _np(kt.grad), rtol=1e-12, atol=1e-11)


def test_conv_1d_is_numpy_convolve():
    """The paper's 1-D listing output(x) = input(x - r.x) * kernel(r.x)
    on one row: numpy's full convolution, shifted by the centring offset kw//2."""
    g = np.random.default_rng(3)
    sig, ker = g.standard_normal(23), g.standard_normal(5)
    y = oracle.conv_fwd(sig.reshape(1, 1, 1, -1), ker.reshape(1, 1, 1, -1)).ravel()
    np.testing.assert_allclose(y, np.convolve(sig, ker, "full")[2:2 + 23], rtol=1e-13, atol=1e-13)


def test_conv_closed_forms():
    """Delta kernel (identity across channels at the centre tap): y = x, dx = dy,
    dk[co,ci,centre] = <dy_co, x_ci>.  A one-tap kernel at r = (0, 0) reads x at
    (y + ph, x + pw) and at r = (2, 2) at (y - 1, x - 1), with zero fill."""
    N, C, H, W = 2, 3, 7, 8
    x, _, dy = _conv_case(N, C, C, H, W, 3, 3, seed=5)
    k = np.zeros((C, C, 3, 3))
    for c in range(C):
        k[c, c, 1, 1] = 1.0
    np.testing.assert_allclose(oracle.conv_fwd(x, k), x, rtol=0, atol=1e-15)
    dx, dk = oracle.conv_bwd(x, k, dy)
    np.testing.assert_allclose(dx, dy, rtol=0, atol=1e-15)
    np.testing.assert_allclose(dk[:, :, 1, 1], np.einsum("nohw,nihw->oi", dy, x), rtol=1e-12, atol=1e-12)
    k1 = np.zeros((1, 1, 3, 3))
    k1[0, 0, 0, 0] = 1.0
    y = oracle.conv_fwd(x[:, :1], k1)
    np.testing.assert_allclose(y[:, 0, :-1, :-1], x[:, 0, 1:, 1:], rtol=0, atol=0)
    assert np.all(y[:, 0, -1, :] == 0) and np.all(y[:, 0, :, -1] == 0)
    k2 = np.zeros((1, 1, 3, 3))
    k2[0, 0, 2, 2] = 1.0
    y = oracle.conv_fwd(x[:, :1], k2)
    np.testing.assert_allclose(y[:, 0, 1:, 1:], x[:, 0, :-1, :-1], rtol=0, atol=0)
    assert np.all(y[:, 0, 0, :] == 0) and np.all(y[:, 0, :, 0] == 0)


@pytest.mark.parametrize("ks", [(2, 2), (4, 3), (3, 3)])
def test_conv_adjoint_identity_and_bilinearity(ks):
    """<conv(x, k), g> = <x, dx(g)> = <k, dk(g)> (the layer is linear in x and in k),
    including even kernel sizes, which no library pin covers."""
    kh, kw = ks
    x, k, dy = _conv_case(2, 3, 2, 9, 6, kh, kw, seed=7)
    y = oracle.conv_fwd(x, k)
    dx, dk = oracle.conv_bwd(x, k, dy)
    lhs = float((y * dy).sum())
    assert abs(lhs - float((x * dx).sum())) <= 1e-12 * max(1.0, abs(lhs))
    assert abs(lhs - float((k * dk).sum())) <= 1e-12 * max(1.0, abs(lhs))


def test_conv_brute_force_operator_matrix():
    """dx = M^T dy with M built column by column from forward calls on basis inputs
    (even 2 x 4 kernel, non-square image, 2 -> 3 channels)."""
    N, Ci, Co, H, W, kh, kw = 1, 2, 3, 4, 5, 2, 4
    _, k, dy = _conv_case(N, Ci, Co, H, W, kh, kw, seed=9)
    n_in = Ci * H * W
    M = np.zeros((Co * H * W, n_in))
    for j in range(n_in):
        e = np.zeros(n_in)
        e[j] = 1.0
        M[:, j] = oracle.conv_fwd(e.reshape(1, Ci, H, W), k).ravel()
    dx, _ = oracle.conv_bwd(np.zeros((N, Ci, H, W)), k, dy)
    np.testing.assert_allclose(dx.ravel(), M.T @ dy.ravel(), rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- checkpointing study (§8(f) f4)
@pytest.mark.parametrize("ks", [(1, 5), (3, 5), (2, 2)])
def test_convloss_grad_vs_torch_autograd(ks):
    """d_in of sum (conv(in, k) - target)^2 = torch autograd of the
    same loss built from conv2d with the flipped kernel (even kernels: asymmetric pad)."""
    kh, kw = ks
    g = np.random.default_rng(11)
    N, H, W = 2, 13, 17
    inp, k, tgt = g.standard_normal((N, H, W)), g.standard_normal((kh, kw)), g.standard_normal((N, H, W))
    it = torch.tensor(inp[:, None], requires_grad=True)
    # y[y,x] = sum_r in[y - ry + kh//2, x - rx + kw//2] k[r]: pad top kh//2, bottom kh-1-kh//2
    pt = F.pad(it, (kw - 1 - kw // 2, kw // 2, kh - 1 - kh // 2, kh // 2))
    conv = F.conv2d(pt, torch.tensor(k).flip(0, 1)[None, None])
    loss = ((conv[:, 0] - torch.tensor(tgt)) ** 2).sum()
    loss.backward()
    np.testing.assert_allclose(oracle.convloss_grad(inp, k, tgt), _np(it.grad)[:, 0], rtol=1e-12, atol=1e-11)


def test_upsample4_vs_torch():
    """output(x) = input(x/4) is nearest upsampling by 4; its adjoint
    sums each 4 x 4 block (torch autograd)."""
    g = np.random.default_rng(12)
    x, dy = g.standard_normal((2, 3, 5, 7)), g.standard_normal((2, 3, 20, 28))
    xt = torch.tensor(x, requires_grad=True)
    yt = F.interpolate(xt, scale_factor=4, mode="nearest")
    yt.backward(torch.tensor(dy))
    np.testing.assert_array_equal(oracle.upsample4_fwd(x), _np(yt))
    np.testing.assert_allclose(oracle.upsample4_bwd(dy), _np(xt.grad), rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(oracle.upsample4_bwd(dy), dy.reshape(2, 3, 5, 4, 7, 4).sum(axis=(3, 5)),
                               rtol=1e-14, atol=1e-14)


# --------------------------------------------------------------------------- STN variants (§8(f) f3)
def _rand_theta(N, rows, seed):
    g = np.random.default_rng(seed)
    th = np.zeros((N, rows, rows + 1))
    for n in range(N):
        th[n, :, :rows] = np.eye(rows) * g.uniform(0.8, 1.2) + g.uniform(-0.25, 0.25, (rows, rows))
        th[n, :, rows] = g.uniform(-0.2, 0.2, rows)
    return th


@pytest.mark.parametrize("ac", [True, False])
def test_stn_bicubic_vs_torch(ac):
    """Bicubic STN = torch affine_grid + grid_sample(mode='bicubic', zeros) in fp64,
    forward and autograd d_input / d_theta ("changing the interpolation
    scheme")."""
    g = np.random.default_rng(21)
    N, C, H, W, Ho, Wo = 2, 3, 11, 13, 9, 10
    x, dy = g.standard_normal((N, C, H, W)), g.standard_normal((N, C, Ho, Wo))
    th = _rand_theta(N, 2, 22)
    xt, tt = torch.tensor(x, requires_grad=True), torch.tensor(th, requires_grad=True)
    grid = F.affine_grid(tt, (N, C, Ho, Wo), align_corners=ac)
    yt = F.grid_sample(xt, grid, mode="bicubic", padding_mode="zeros", align_corners=ac)
    yt.backward(torch.tensor(dy))
    np.testing.assert_allclose(oracle.stn_bicubic_fwd(x, th, Ho, Wo, ac), _np(yt), rtol=1e-11, atol=1e-12)
    dx, dth = oracle.stn_bicubic_bwd(x, th, dy, ac)
    np.testing.assert_allclose(dx, _np(xt.grad), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dth, _np(tt.grad), rtol=1e-10, atol=1e-10)


def test_stn_bicubic_identity_interpolates():
    """Keys' kernel interpolates: identity theta (align_corners=1) reproduces x up to the
    rounding of the normalisation round trip."""
    x = np.random.default_rng(23).standard_normal((1, 2, 8, 9))
    th = np.array([[[1.0, 0, 0], [0, 1.0, 0]]])
    np.testing.assert_allclose(oracle.stn_bicubic_fwd(x, th), x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("ac", [True, False])
def test_stn3d_vs_torch(ac):
    """Volumetric STN = torch 5-D affine_grid + trilinear grid_sample (zeros) in fp64,
    forward and autograd ("interpolating over more dimensions")."""
    g = np.random.default_rng(24)
    N, C, D, H, W, Do, Ho, Wo = 2, 2, 5, 6, 7, 4, 6, 5
    x, dy = g.standard_normal((N, C, D, H, W)), g.standard_normal((N, C, Do, Ho, Wo))
    th = _rand_theta(N, 3, 25)
    xt, tt = torch.tensor(x, requires_grad=True), torch.tensor(th, requires_grad=True)
    grid = F.affine_grid(tt, (N, C, Do, Ho, Wo), align_corners=ac)
    yt = F.grid_sample(xt, grid, mode="bilinear", padding_mode="zeros", align_corners=ac)
    yt.backward(torch.tensor(dy))
    np.testing.assert_allclose(oracle.stn3d_fwd(x, th, (Do, Ho, Wo), ac), _np(yt), rtol=1e-11, atol=1e-12)
    dx, dth = oracle.stn3d_bwd(x, th, dy, ac)
    np.testing.assert_allclose(dx, _np(xt.grad), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dth, _np(tt.grad), rtol=1e-10, atol=1e-10)


def test_stn3d_reduces_to_2d_on_one_slice():
    """On a one-slice volume (align_corners=0) a 3-D theta that leaves z alone samples
    the slice exactly (f_z = 0): the 2-D STN of that slice (cross-layer invariant)."""
    g = np.random.default_rng(26)
    x = g.standard_normal((1, 2, 1, 9, 11))
    th2 = _rand_theta(1, 2, 27)
    th3 = np.zeros((1, 3, 4))
    th3[0, :2, :2], th3[0, :2, 3] = th2[0, :, :2], th2[0, :, 2]
    th3[0, 2, 2] = 1.0
    y3 = oracle.stn3d_fwd(x, th3, (1, 9, 11), align_corners=False)
    y2 = oracle.stn_fwd(x[:, :, 0], th2, align_corners=False)
    np.testing.assert_allclose(y3[:, :, 0], y2, rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- kink diagnostics
def test_kink_counts():
    """SURVEY 8(c) diagnostic: identity theta (align_corners=1) and zero flow put every
    sample exactly on the grid (2 axes x pixels); the quarter-pixel theta puts none there;
    guide values k/D + 1/(2D) sit exactly on the guide-axis kink."""
    th = np.array([[[1.0, 0, 0], [0, 1.0, 0]]] * 2)
    assert oracle.stn_kinks(th, 8, 9) == 2 * 2 * 8 * 9
    q = np.array([[[1.0, 0, 0.5 / 8], [0, 1.0, 0.5 / 7]]])
    assert oracle.stn_kinks(q, 8, 9) == 0
    assert oracle.warp_kinks(np.zeros((1, 2, 5, 6))) == 2 * 30
    assert oracle.warp_kinks(np.full((1, 2, 5, 6), 0.25)) == 0
    g = (np.arange(8)[None, None, :] + 0.5) / 8 * np.ones((1, 3, 8))
    assert oracle.bslice_kinks(g, 8) == 24
    assert oracle.bslice_kinks(g + 0.01, 8) == 0


# --------------------------------------------------------------------------- Lanczos-3 STN (§8(f) f3)
def test_lanczos3_kernel_is_numpy_sinc():
    """L(x) = sinc(x) sinc(x/3) on |x| < 3 (numpy's normalised sinc), 0 outside; L' matches
    a central difference of numpy's expression."""
    for x in np.linspace(-3.5, 3.5, 141):
        ref = np.sinc(x) * np.sinc(x / 3) if abs(x) < 3 else 0.0
        assert abs(oracle.lanczos3(x) - ref) <= 1e-14
        if 1e-3 < abs(x) < 2.999:
            h = 1e-6
            fd = (np.sinc(x + h) * np.sinc((x + h) / 3) - np.sinc(x - h) * np.sinc((x - h) / 3)) / (2 * h)
            assert abs(oracle.dlanczos3(x) - fd) <= 1e-8


def test_stn_lanczos_identity_and_adjoint():
    """Lanczos interpolates (L(0) = 1, L(k) = 0): identity theta reproduces x; the adjoint
    is the transpose (adjoint identity, brute-force operator matrix)."""
    g = np.random.default_rng(41)
    x = g.standard_normal((1, 2, 9, 11))
    th = np.array([[[1.0, 0, 0], [0, 1.0, 0]]])
    np.testing.assert_allclose(oracle.stn_lanczos_fwd(x, th), x, rtol=0, atol=1e-12)
    th = _rand_theta(1, 2, 42)
    C, H, W = 1, 6, 7
    n_in = C * H * W
    M = np.zeros((C * H * W, n_in))
    for j in range(n_in):
        e = np.zeros(n_in)
        e[j] = 1.0
        M[:, j] = oracle.stn_lanczos_fwd(e.reshape(1, C, H, W), th).ravel()
    dy = g.standard_normal((1, C, H, W))
    dx, _ = oracle.stn_lanczos_bwd(np.zeros((1, C, H, W)), th, dy)
    np.testing.assert_allclose(dx.ravel(), M.T @ dy.ravel(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("ac", [True, False])
def test_stn_lanczos_fwd_brute_force_all_pixels(ac):
    """Independent pin of the 6-tap window (R13): the forward
    equals sum over EVERY image pixel (l, k) of L(iy - l) L(ix - k) X[l, k], with
    L(t) = numpy sinc(t) sinc(t/3) on |t| < 3 -- no window at all, so an off-by-one tap
    window (e.g. floor-3 .. floor+2) would drop a nonzero term and fail.  Random theta,
    zoom and shift: sample points off the integers, partly outside the image (zeros)."""
    g = np.random.default_rng(45)
    N, C, H, W, Ho, Wo = 2, 2, 9, 11, 7, 8
    x = g.standard_normal((N, C, H, W))
    th = np.array([[[1.0, 0, 0], [0, 1.0, 0]]] * N) + g.normal(0, 0.25, (N, 2, 3))

    def L(t):
        return np.where(np.abs(t) < 3, np.sinc(t) * np.sinc(t / 3), 0.0)

    if ac:
        xt = -1 + 2 * np.arange(Wo) / (Wo - 1)
        yt = -1 + 2 * np.arange(Ho) / (Ho - 1)
    else:
        xt = (2 * np.arange(Wo) + 1) / Wo - 1
        yt = (2 * np.arange(Ho) + 1) / Ho - 1
    ref = np.zeros((N, C, Ho, Wo))
    ls, ks = np.arange(H), np.arange(W)
    offint = []
    for n in range(N):
        for i in range(Ho):
            for j in range(Wo):
                gx = th[n, 0, 0] * xt[j] + th[n, 0, 1] * yt[i] + th[n, 0, 2]
                gy = th[n, 1, 0] * xt[j] + th[n, 1, 1] * yt[i] + th[n, 1, 2]
                ix = (gx + 1) * (W - 1) / 2 if ac else ((gx + 1) * W - 1) / 2
                iy = (gy + 1) * (H - 1) / 2 if ac else ((gy + 1) * H - 1) / 2
                offint.append(min(abs(ix - round(ix)), abs(iy - round(iy))) > 1e-3)
                wgt = np.outer(L(iy - ls), L(ix - ks))  # H x W, every pixel
                ref[n, :, i, j] = (x[n] * wgt).sum(axis=(1, 2))
    assert np.mean(offint) > 0.9  # L is continuous; off-integer points see all 6 taps
    y = oracle.stn_lanczos_fwd(x, th, Ho, Wo, ac)
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


def test_stn_lanczos_theta_central_fd():
    """d_theta vs central finite differences of <y(theta), dy> with
    sample coordinates kept away from the kernel's kinks (integers)."""
    g = np.random.default_rng(43)
    x, dy = g.standard_normal((1, 2, 10, 12)), g.standard_normal((1, 2, 8, 9))
    th = _rand_theta(1, 2, 44)
    _, dth = oracle.stn_lanczos_bwd(x, th, dy)
    h = 1e-6
    for r in range(2):
        for c in range(3):
            tp, tm = th.copy(), th.copy()
            tp[0, r, c] += h
            tm[0, r, c] -= h
            fd = ((oracle.stn_lanczos_fwd(x, tp, 8, 9) - oracle.stn_lanczos_fwd(x, tm, 8, 9)) * dy).sum() / (2 * h)
            assert abs(dth[0, r, c] - fd) <= 1e-5 * max(1.0, abs(fd))
