"""Tolerance comparator for CUDA-vs-oracle parity.

Elementwise:  |g - r| <= rtol*|r| + atol*s,  s = max(1, rms(r)) over the tensor.
Forward outputs: rtol 1e-5, atol 1e-6.  Gradients: rtol 1e-4, atol 1e-6
(BASELINE.json north_star "rel 1e-5 fwd, rel 1e-4 (abs 1e-6) grads"; the
rms scaling of the absolute floor is reading T of SURVEY.md 8(c)).
"""
import numpy as np

FWD = dict(rtol=1e-5, atol=1e-6)
GRAD = dict(rtol=1e-4, atol=1e-6)


def compare(g, r, rtol, atol):
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    if r.size == 0:
        return {"ok": True, "n_fail": 0, "max_ratio": 0.0, "normwise": 0.0, "n": 0}
    s = max(1.0, float(np.sqrt(np.mean(r * r))))
    err = np.abs(g - r)
    bound = rtol * np.abs(r) + atol * s
    ratio = err / bound
    nr = float(np.linalg.norm(r))
    return {
        "ok": bool(np.all(err <= bound)),
        "n_fail": int(np.count_nonzero(err > bound)),
        "max_ratio": float(ratio.max()),
        "normwise": float(np.linalg.norm(g - r) / nr) if nr > 0 else float(np.linalg.norm(g - r)),
        "n": int(r.size),
    }


def assert_close(g, r, kind, what=""):
    tol = FWD if kind == "fwd" else GRAD
    rep = compare(g, r, **tol)
    assert rep["ok"], f"{what}: {rep}"
    return rep
