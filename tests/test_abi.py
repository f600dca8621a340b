"""C-ABI boundary checks that need no GPU: the library builds for sm_100a, loads,
exports every symbol include/rsgrad.h declares, and validates arguments
(status codes + rsgrad_last_error) before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1904_12228_b200 import _build, rsgrad

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsgrad.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w ]+?\*?\s*\b(\w+)\s*\(", txt, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while", "defined")))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("stn_fwd", "stn_bwd", "warp_fwd", "warp_bwd", "bslice_fwd", "bslice_bwd",
              "rsgrad_bwd_workspace_bytes", "rsgrad_last_error"):
        assert f in names, names


def test_library_builds_and_exports_every_declared_symbol():
    path = _build.build()
    assert os.path.exists(path)
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    L = ctypes.CDLL(path)
    for f in declared_functions():
        assert hasattr(L, f)


def test_sass_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", _build.build()], text=True)
    assert "sm_100a" in out


def test_version_string():
    assert "sm_100a" in rsgrad.version()


def _o(**kw):
    d = dict(align_corners=1, padding=0, algo=0, deterministic=0)
    d.update(kw)
    return rsgrad.RsOpts(**d)


def test_validation_null_and_shape():
    L = rsgrad.lib()
    o = _o()
    fake = ctypes.c_void_p(0x1000)
    st = L.stn_fwd(None, fake, 1, 1, 4, 4, 4, 4, ctypes.byref(o), fake, None)
    assert st == -1 and b"required" in L.rsgrad_last_error()
    st = L.stn_fwd(fake, fake, 1, 0, 4, 4, 4, 4, ctypes.byref(o), fake, None)
    assert st == -2
    st = L.stn_fwd(fake, fake, 1, 1, 4, 4, 1, 4, ctypes.byref(o), fake, None)
    assert st == -2 and b"align_corners" in L.rsgrad_last_error()
    st = L.warp_fwd(fake, None, 1, 1, 4, 4, ctypes.byref(o), fake, None)
    assert st == -1
    st = L.bslice_fwd(fake, fake, fake, 1, 4, 4, 0, 2, 2, ctypes.byref(o), fake, None)
    assert st == -2


def test_validation_flags():
    L = rsgrad.lib()
    fake = ctypes.c_void_p(0x1000)
    bad = _o(padding=7)
    assert L.warp_fwd(fake, fake, 1, 1, 4, 4, ctypes.byref(bad), fake, None) == -4
    # GATHER is refused for warp d_input and for STN with border padding
    g = _o(algo=1)
    assert L.warp_bwd(fake, fake, fake, 1, 1, 4, 4, ctypes.byref(g), fake, None, None, 0, None) == -4
    gb = _o(algo=1, padding=1)
    assert L.stn_bwd(fake, fake, fake, 1, 1, 4, 4, 4, 4, ctypes.byref(gb), fake, None, None, 0,
                     None) == -4
    det = _o(algo=3, deterministic=1)
    assert L.bslice_bwd(fake, fake, fake, fake, 1, 64, 64, 8, 4, 4, ctypes.byref(det), fake, None,
                        None, None, 0, None) == -4


def test_workspace_sizes():
    # STN: per-block fp64 d_theta partials + coordinate tables + one channel plane of 64-bit
    # fixed-point accumulators (AUTO's exact scatter of high fan-in fallback samples)
    assert rsgrad.workspace_bytes(0, 4, 16, 512, 512, 512, 512) >= 8 * 512 * 512
    # warp AUTO: room for the fixed-point recompute of heavy (collapsing) samples + flags
    assert rsgrad.workspace_bytes(1, 8, 3, 384, 512) >= 8 * 3 * 384 * 512 + 4 * 8
    # deterministic=1: + one sample of 64-bit fixed-point accumulators (det.cuh)
    det = rsgrad._opts(deterministic=True)
    assert rsgrad.workspace_bytes(1, 8, 3, 384, 512, opts=det) >= 8 * 3 * 384 * 512
    assert (rsgrad.workspace_bytes(0, 4, 16, 512, 512, 512, 512, opts=det)
            >= rsgrad.workspace_bytes(0, 4, 16, 512, 512, 512, 512) + 8 * 15 * 512 * 512)
    # bslice tiled path: one partial per (dual cell, corner, z, q) + the per-call
    # dual-cell bounds table (Gh + Gw + 4 ints)
    ws = rsgrad.workspace_bytes(2, 4, 3, 1024, 1024, D=8, Gh=16, Gw=16)
    assert ws == 4 * 17 * 17 * 4 * 8 * 12 * 4 + 4 * (16 + 16 + 4)
    # too-fine grid => atomic path: only the bounds table (GATHER's node walk uses it);
    # deterministic=1: the fixed-point d_grid
    assert rsgrad.workspace_bytes(2, 1, 3, 16, 16, D=8, Gh=16, Gw=16) == 4 * (16 + 16 + 4)
    assert rsgrad.workspace_bytes(2, 1, 3, 16, 16, D=8, Gh=16, Gw=16,
                                  opts=rsgrad._opts(deterministic=True)) >= 8 * 12 * 8 * 16 * 16
    assert rsgrad.workspace_bytes(9, 1) == 0


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = torch.zeros(1, 1, 4, 4)
    th = torch.zeros(1, 2, 3)
    with pytest.raises(rsgrad.RsgradError):
        rsgrad.stn_fwd(x, th)


def test_conv_validation():
    """conv_* argument checks that need no GPU: NULLs, non-positive dims, kernel size."""
    L = rsgrad.lib()
    fake = ctypes.c_void_p(0x1000)
    o = _o()
    assert L.conv_fwd(None, fake, 1, 1, 1, 4, 4, 3, 3, ctypes.byref(o), fake, None) == -1
    assert L.conv_fwd(fake, fake, 1, 0, 1, 4, 4, 3, 3, ctypes.byref(o), fake, None) == -2
    assert L.conv_fwd(fake, fake, 1, 1, 1, 4, 4, 9, 3, ctypes.byref(o), fake, None) == -2
    assert L.conv_bwd(fake, fake, fake, 1, 1, 1, 4, 4, 3, 8, ctypes.byref(o), fake, None, None, 0, None) == -2
    # d_kernel tile in shared memory: Ci <= 68 at 3x3 with Co = 16 (include/rsgrad.h)
    assert L.conv_fwd(fake, fake, 1, 69, 16, 8, 8, 3, 3, ctypes.byref(o), fake, None) == -2
    assert L.conv_fwd(fake, fake, 1, 68, 16, 8, 8, 3, 3, ctypes.byref(o), fake, None) != -2
    # d_kernel partials: one per persistent block (<= 296) x Co x Ci x kh x kw doubles
    assert rsgrad.workspace_bytes(3, 16, 16, 256, 256, D=16, Gh=3, Gw=3) == 296 * 16 * 16 * 9 * 8
