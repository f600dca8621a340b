"""paper_1904_12228_b200 — B200-native forward + adjoint kernels for the resampling
layers of gradient Halide's "Custom Neural Network Layers" (arXiv 1904.12228,
PAPER.md:11-42): spatial transformer, FlowNet 2.0 warp, HDRNet bilateral slice.

The compute lives in ``librsgrad.so`` (C ABI: ``include/rsgrad.h``); this package
is the thin ctypes binding (``rsgrad``) plus autograd wrappers.
"""
from .rsgrad import (  # noqa: F401
    BilateralSlice,
    FlowWarp,
    RsgradError,
    SpatialTransformer,
    bslice_bwd,
    bslice_fwd,
    launch_count,
    lib,
    stn_bwd,
    stn_fwd,
    version,
    warp_bwd,
    warp_fwd,
    workspace_bytes,
)

__all__ = [
    "stn_fwd", "stn_bwd", "warp_fwd", "warp_bwd", "bslice_fwd", "bslice_bwd",
    "SpatialTransformer", "FlowWarp", "BilateralSlice", "RsgradError", "lib", "version",
    "launch_count", "workspace_bytes",
]
