"""The C-ABI calls captured into a CUDA graph (include/rsgrad.h "Graphs") and replayed on
fresh inputs copied into the captured buffers: every replay matches the fp64 oracle
within the north star's tolerance (tests/_tol.py), like the eager calls.  Covers the
multi-kernel backward sequences (STN prep / lean / dtheta / finalize, warp strip +
fixed-point rescue of heavy samples, bslice tiles + gathers) and the workspace that
the binding allocates inside the capture."""
import pytest
import torch

import oracle
import synth
from paper_1904_12228_b200 import rsgrad
from _tol import assert_close
from test_parity_gpu import _collapse_flow

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().double().numpy()


def _graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def _load(bufs, inp):
    for k, b in bufs.items():
        b.copy_(inp[k])


@pytest.mark.parametrize("padding,W,mode", [("zeros", 70, "auto"), ("border", 70, "auto"), ("zeros", 72, "auto"),
                                            ("zeros", 72, "prep")])
def test_stn_graph_replay(cuda_device, monkeypatch, padding, W, mode):
    """W = 72 (rows 16-B aligned): the three-launch path with the d_theta tiles forked onto
    the library side stream inside the capture; mode prep: the prep / finalize kernels."""
    if mode == "prep":
        monkeypatch.setenv("RSGRAD_STN_PREP", "1")
    N, C, H = 3, 5, 61
    mk = lambda n0: synth.stn_inputs(N, C, H, W, cfg=1, n0=n0)  # noqa: E731
    bufs = {k: v.to(cuda_device).contiguous() for k, v in mk(0).items()}
    y = torch.empty_like(bufs["dy"])
    dx, dth = torch.empty_like(bufs["x"]), torch.empty_like(bufs["theta"])
    border = padding == "border"

    def step():
        rsgrad.stn_fwd(bufs["x"], bufs["theta"], padding=padding, out=y)
        rsgrad.stn_bwd(bufs["x"], bufs["theta"], bufs["dy"], padding=padding, out=(dx, dth))

    g = _graph(step)
    for n0 in (7, 19):
        inp = mk(n0)
        _load(bufs, inp)
        g.replay()
        torch.cuda.synchronize()
        x, th, dy = (inp[k].double().numpy() for k in ("x", "theta", "dy"))
        assert_close(_np(y), oracle.stn_fwd(x, th, H, W, True, border), "fwd", "y")
        rdx, rdth = oracle.stn_bwd(x, th, dy, True, border)
        assert_close(_np(dx), rdx, "grad", "dx")
        assert_close(_np(dth), rdth, "grad", "dtheta")


@pytest.mark.parametrize("flows", [("smooth", "collapse", "smooth"), ("collapse", "stress", "collapse")])
def test_warp_graph_replay(cuda_device, flows):
    """The heavy-sample flags live in the captured workspace and the tag is fixed at
    capture: a replay after a collapsing flow must still be exact (flags are cleared by
    the fixed-point pass) and a collapsing replay must still be rescued."""
    N, C, H, W = 2, 3, 96, 128
    def mk(n0, fl):
        inp = synth.warp_inputs(N, C, H, W, cfg=1, flow="smooth" if fl == "collapse" else fl, n0=n0)
        if fl == "collapse":
            inp["flow"] = _collapse_flow(N, H, W)
        return inp

    bufs = {k: v.to(cuda_device).contiguous() for k, v in mk(0, flows[0]).items()}
    y, dx, df = torch.empty_like(bufs["x"]), torch.empty_like(bufs["x"]), torch.empty_like(bufs["flow"])

    def step():
        rsgrad.warp_fwd(bufs["x"], bufs["flow"], padding="border", out=y)
        rsgrad.warp_bwd(bufs["x"], bufs["flow"], bufs["dy"], padding="border", out=(dx, df))

    g = _graph(step)
    for r, fl in enumerate(flows):
        inp = mk(3 + r, fl)
        _load(bufs, inp)
        g.replay()
        torch.cuda.synchronize()
        x, f, dy = (inp[k].double().numpy() for k in ("x", "flow", "dy"))
        assert_close(_np(y), oracle.warp_fwd(x, f, True), "fwd", "y")
        rdx, rdf = oracle.warp_bwd(x, f, dy, True)
        assert_close(_np(dx), rdx, "grad", "dx")
        assert_close(_np(df), rdf, "grad", "dflow")


@pytest.mark.parametrize("grid", [(8, 16, 16), (8, 4, 5)])
def test_bslice_graph_replay(cuda_device, grid):
    N, H, W = 2, 128, 160
    D, Gh, Gw = grid
    mk = lambda n0: synth.bslice_inputs(N, H, W, D, Gh, Gw, cfg=1, grid="iid", n0=n0)  # noqa: E731
    bufs = {k: v.to(cuda_device).contiguous() for k, v in mk(0).items()}
    y = torch.empty_like(bufs["x"])
    dgr, dgd, dx = torch.empty_like(bufs["grid"]), torch.empty_like(bufs["guide"]), torch.empty_like(bufs["x"])

    def step():
        rsgrad.bslice_fwd(bufs["grid"], bufs["guide"], bufs["x"], out=y)
        rsgrad.bslice_bwd(bufs["grid"], bufs["guide"], bufs["x"], bufs["dy"], out=(dgr, dgd, dx))

    g = _graph(step)
    for n0 in (5, 11):
        inp = mk(n0)
        _load(bufs, inp)
        g.replay()
        torch.cuda.synchronize()
        gr, gd, x, dy = (inp[k].double().numpy() for k in ("grid", "guide", "x", "dy"))
        assert_close(_np(y), oracle.bslice_fwd(gr, gd, x), "fwd", "y")
        rgr, rgd, rdx = oracle.bslice_bwd(gr, gd, x, dy)
        assert_close(_np(dx), rdx, "grad", "dx")
        assert_close(_np(dgd), rgd, "grad", "dguide")
        assert_close(_np(dgr), rgr, "grad", "dgrid")
