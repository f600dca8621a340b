"""Build librsgrad.so (all CUDA sources, sm_100a) in-tree with nvcc.

Each .cu is compiled to an object in parallel (build/obj), then linked into
paper_1904_12228_b200/librsgrad.so.  RSGRAD_NVCC_EXTRA (space-separated flags) and
``build(out=...)`` produce A/B variants of the library without touching the default.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shlex
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librsgrad.so")
HEADER = os.path.join(ROOT, "include", "rsgrad.h")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-diag-suppress", "177",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]


def _stale(out: str) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in _deps())


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra=None) -> str:
    out = out or LIB
    if extra is None:
        extra = shlex.split(os.environ.get("RSGRAD_NVCC_EXTRA", ""))
    if not force and not _stale(out):
        return out
    tag = os.path.basename(out).replace(".so", "")
    odir = os.path.join(OBJ, tag)
    os.makedirs(odir, exist_ok=True)
    flags = [*NVCC_FLAGS, *extra] + (["-Xptxas=-v"] if verbose else [])

    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    flagfile = os.path.join(odir, "flags.txt")
    same_flags = os.path.exists(flagfile) and open(flagfile).read() == " ".join(flags)

    def compile_one(src):
        obj = os.path.join(odir, os.path.basename(src).replace(".cu", ".o"))
        if same_flags and not force and os.path.exists(obj):
            t = os.path.getmtime(obj)
            if all(os.path.getmtime(p) <= t for p in [src, *hdrs]):
                return obj
        cmd = [nvcc(), *flags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    with open(flagfile, "w") as f:
        f.write(" ".join(flags))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, out)
    return out
