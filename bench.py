#!/usr/bin/env python
"""bench.py — fwd+bwd throughput of the three resampling layers on B200.

Workload (BASELINE.json configs[4], the configuration the metric is quoted on):
batch 64 at 1024 x 1024 through STN (C=16, theta as configs[1]), FlowNet warp
(C=3, smooth flow) and bilateral slice-apply (grid 16x16x8, 12 coefficients).
One STEP = stn_fwd + stn_bwd + warp_fwd + warp_bwd + bslice_fwd + bslice_bwd
over the rank's shard of the batch (every sample's parameters are its own:
batch sharding, no collective on the data path).  The global batch is fixed
(64), so scaling is strong.

value      = N*H*W pixel positions of the global batch / device time of a step
             (max over ranks), in Mpix/s; each pixel position passes fwd+bwd
             through all three layers.
e2e        = the same step through the C ABI with pinned HOST buffers: the
             library stages every input H2D and every output D2H on the stream.
roofline   = the dominant call of the step: algorithmic bytes (DESIGN.md
             "Algorithmic bytes") / its CUDA-event duration vs MEASURED_PEAKS.json.
cpu_baseline = the fp64 oracle (oracle/) timed on the host cores on one sample of
             each layer (rank 0, N=1 only).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

BATCH, H, W = 64, 1024, 1024
C_STN, C_WARP = 16, 3
D, GH, GW = 8, 16, 16
METRIC = "fwd+bwd Mpix/s per layer and % HBM roofline at 1/2/4/8 B200"
UNIT = "Mpix/s"

# algorithmic bytes per pixel position (compulsory traffic only)
BYTES = {
    ("stn", "fwd"): lambda C: 8 * C, ("stn", "bwd"): lambda C: 12 * C,
    ("warp", "fwd"): lambda C: 8 + 8 * C, ("warp", "bwd"): lambda C: 16 + 12 * C,
    ("bslice", "fwd"): lambda C: 28, ("bslice", "bwd"): lambda C: 44,
}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- distributed
def spawn_ranks(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous), exactly
    as the driver launches it.  Returns only when no re-exec is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist

        if args.dry_run:  # CPU plumbing test: gloo, no device
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available() and not args.dry_run:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, vals):
    """Element-wise MAX over ranks (timings are reported as the slowest rank)."""
    dev = "cpu"
    if world > 1:
        import torch.distributed as dist

        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def shard(world, rank, batch=BATCH):
    per = batch // world
    assert per * world == batch, "global batch must divide the GPU count"
    return rank * per, per


# --------------------------------------------------------------------------- workload
def make_inputs(n0, nb, dev):
    import synth

    s = synth.stn_inputs(nb, C_STN, H, W, cfg=5, device=dev, n0=n0)
    w = synth.warp_inputs(nb, C_WARP, H, W, cfg=5, device=dev, flow="smooth", n0=n0)
    b = synth.bslice_inputs(nb, H, W, D, GH, GW, cfg=5, device=dev, n0=n0)
    return s, w, b


def alloc_outputs(s, w, b, host=False):
    def e(ref):
        if host:
            return torch.empty(ref.shape, dtype=torch.float32, pin_memory=True)
        return torch.empty_like(ref)

    nb = s["x"].shape[0]
    return {
        "stn_y": e(s["dy"]), "stn_dx": e(s["x"]), "stn_dth": e(s["theta"]),
        "warp_y": e(w["dy"]), "warp_dx": e(w["x"]), "warp_df": e(w["flow"]),
        "bs_y": e(b["dy"]), "bs_dgr": e(b["grid"]), "bs_dgd": e(b["guide"]), "bs_dx": e(b["x"]),
        "_nb": nb,
    }


def config_dict(world):
    return {"workload": "configs[4]: batch 64 @ 1024x1024 per layer (STN C=16 | warp C=3 smooth "
                        "flow | bslice grid 16x16x8x12), one step = fwd+bwd of all three",
            "global_batch": BATCH, "H": H, "W": W, "per_rank_batch": BATCH // world,
            "parallelism": f"batch-shard x{world}, no data-path collective",
            "l2": "inputs > L2 (4.3 GB STN tensors), no flush between steps"}


def step_calls(rs, s, w, b, o, sync=True):
    """The six C-ABI calls of one step, as (name, thunk)."""
    return [
        ("stn_fwd", lambda: rs.stn_fwd(s["x"], s["theta"], out=o["stn_y"], sync=sync)),
        ("stn_bwd", lambda: rs.stn_bwd(s["x"], s["theta"], s["dy"], out=(o["stn_dx"], o["stn_dth"]),
                                       sync=sync)),
        ("warp_fwd", lambda: rs.warp_fwd(w["x"], w["flow"], out=o["warp_y"], sync=sync)),
        ("warp_bwd", lambda: rs.warp_bwd(w["x"], w["flow"], w["dy"], out=(o["warp_dx"], o["warp_df"]),
                                         sync=sync)),
        ("bslice_fwd", lambda: rs.bslice_fwd(b["grid"], b["guide"], b["x"], out=o["bs_y"], sync=sync)),
        ("bslice_bwd", lambda: rs.bslice_bwd(b["grid"], b["guide"], b["x"], b["dy"],
                                             out=(o["bs_dgr"], o["bs_dgd"], o["bs_dx"]), sync=sync)),
    ]


CALL_BYTES = {
    "stn_fwd": BYTES[("stn", "fwd")](C_STN), "stn_bwd": BYTES[("stn", "bwd")](C_STN),
    "warp_fwd": BYTES[("warp", "fwd")](C_WARP), "warp_bwd": BYTES[("warp", "bwd")](C_WARP),
    "bslice_fwd": BYTES[("bslice", "fwd")](0), "bslice_bwd": BYTES[("bslice", "bwd")](0),
}


# --------------------------------------------------------------------------- paper shapes
def flush_l2(buf):
    buf.add_(1.0)


def paper_cases(rs, dev):
    """configs[1..3] (+ the paper's 32x32x8 and 2048^2 bslice grids): (name, layer, C, P,
    fwd thunk, bwd thunk) with inputs and outputs resident on dev."""
    import synth

    cases = [
        ("stn_4x16x512x512", "stn", C_STN, synth.stn_inputs(4, 16, 512, 512, cfg=2, device=dev)),
        ("warp_8x3x384x512_smooth", "warp", 3, synth.warp_inputs(8, 3, 384, 512, cfg=3, device=dev)),
        ("warp_8x3x384x512_stress", "warp", 3,
         synth.warp_inputs(8, 3, 384, 512, cfg=3, device=dev, flow="stress")),
        ("bslice_4x1024x1024_g16x16x8", "bslice", 3,
         synth.bslice_inputs(4, 1024, 1024, 8, 16, 16, cfg=4, device=dev)),
        ("bslice_4x1024x1024_g32x32x8", "bslice", 3,
         synth.bslice_inputs(4, 1024, 1024, 8, 32, 32, cfg=4, device=dev)),
        # §8(f) f2: the paper's high-resolution case (batch unstated, 4 as above)
        ("bslice_4x2048x2048_g64x64x8", "bslice", 3,
         synth.bslice_inputs(4, 2048, 2048, 8, 64, 64, cfg=4, device=dev)),
    ]
    res = []
    for name, layer, C, i in cases:
        if layer == "stn":
            o = (torch.empty_like(i["x"]), torch.empty_like(i["theta"]))
            y = torch.empty_like(i["dy"])
            fwd = lambda i=i, y=y: rs.stn_fwd(i["x"], i["theta"], out=y)  # noqa: E731
            bwd = lambda i=i, o=o: rs.stn_bwd(i["x"], i["theta"], i["dy"], out=o)  # noqa: E731
            P = i["x"].shape[0] * 512 * 512
        elif layer == "warp":
            o = (torch.empty_like(i["x"]), torch.empty_like(i["flow"]))
            y = torch.empty_like(i["x"])
            fwd = lambda i=i, y=y: rs.warp_fwd(i["x"], i["flow"], out=y)  # noqa: E731
            bwd = lambda i=i, o=o: rs.warp_bwd(i["x"], i["flow"], i["dy"], out=o)  # noqa: E731
            P = 8 * 384 * 512
        else:
            o = (torch.empty_like(i["grid"]), torch.empty_like(i["guide"]), torch.empty_like(i["x"]))
            y = torch.empty_like(i["x"])
            fwd = lambda i=i, y=y: rs.bslice_fwd(i["grid"], i["guide"], i["x"], out=y)  # noqa: E731
            bwd = lambda i=i, o=o: rs.bslice_bwd(i["grid"], i["guide"], i["x"], i["dy"], out=o)  # noqa: E731
            P = i["x"].shape[0] * i["x"].shape[2] * i["x"].shape[3]
        res.append((name, layer, C, P, fwd, bwd))
    return res


def capture(fn):
    """fn's launches captured once into a CUDA graph (the C-ABI calls are capture-safe:
    stream-ordered work only); returns the replay thunk."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm: lazy attributes, allocator
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


def paper_shapes(rs, peak, reps=25, skip=5):
    """configs[1..3] (+ the paper's 32x32x8 grid), each call timed alone after an L2 flush,
    launched eagerly and as one CUDA-graph replay (the per-kernel launch
    tails of a multi-kernel call at these small shapes)."""
    dev = torch.device("cuda")
    fl = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 2x L2
    out = {}
    for name, layer, C, P, fwd, bwd in paper_cases(rs, dev):
        gf, gb = capture(fwd), capture(bwd)
        times = {k: [] for k in ("fwd", "bwd", "fwd_graph", "bwd_graph")}
        for rep in range(reps):
            for kind, fn in (("fwd", fwd), ("bwd", bwd), ("fwd_graph", gf), ("bwd_graph", gb)):
                flush_l2(fl)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if rep >= skip:
                    times[kind].append(e0.elapsed_time(e1) * 1e-3)
        t = {k: statistics.median(v) for k, v in times.items()}
        tf, tb = min(t["fwd"], t["fwd_graph"]), min(t["bwd"], t["bwd_graph"])
        bf, bb = BYTES[(layer, "fwd")](C) * P, BYTES[(layer, "bwd")](C) * P
        out[name] = {
            "fwd_us": round(t["fwd"] * 1e6, 2), "bwd_us": round(t["bwd"] * 1e6, 2),
            "fwd_us_graph": round(t["fwd_graph"] * 1e6, 2), "bwd_us_graph": round(t["bwd_graph"] * 1e6, 2),
            "fwd_bwd_mpix_s": round(P / (tf + tb) / 1e6, 1),
            "bwd_mpix_s": round(P / tb / 1e6, 1),
            "fwd_roofline_frac": round(bf / tf / 1e9 / peak, 3),
            "bwd_roofline_frac": round(bb / tb / 1e9 / peak, 3),
        }
    del fl
    return {"l2": f"flushed (256 MB write) before every call; median of {reps - skip}; eager and "
                  "CUDA-graph replay (*_graph), fractions and Mpix/s from the faster of the two",
            "cases": out}


# --------------------------------------------------------------------------- §8(f) NEXT rows
def fp32_peak_tflops():
    """FP32 FMA peak from the unit counts and clock (B200_PROFILING.md: 148 SMs x 128
    FP32 lanes x 2 flop/FMA x max SM clock)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f)["sm_max_mhz"])
    except Exception:  # noqa: BLE001
        mhz = 1965.0
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def next_rows(rs, peak):
    """SURVEY §8(f) rows at the paper's shapes, each call timed alone after an L2 flush
    (median of 10).  f1: the conv layer of PAPER.md:733 (16 x 16 x 256 x 256, 3 x 3
    chosen: the paper does not state the kernel size), d_input by the converted gather
    vs the atomic scatter; the paper's 68 ms / 6 ms (GPU unstated) are context only."""
    dev = torch.device("cuda")
    fl = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def med(fn, reps=10):
        fn()
        ts = []
        for _ in range(reps):
            flush_l2(fl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(ts)

    out = {}
    g = torch.Generator(device=dev).manual_seed(733)
    N, C, H, W, k = 16, 16, 256, 256, 3
    x = torch.randn(N, C, H, W, device=dev, generator=g)
    kk = torch.randn(C, C, k, k, device=dev, generator=g) / (C * k * k) ** 0.5
    dy = torch.randn(N, C, H, W, device=dev, generator=g)
    y, dx, dk = torch.empty_like(x), torch.empty_like(x), torch.empty_like(kk)
    tf = med(lambda: rs.conv_fwd(x, kk, out=y))
    tg = med(lambda: rs.conv_bwd(x, kk, dy, out=(dx, dk)))
    tdx = med(lambda: rs.conv_bwd(x, kk, dy, need_dk=False, out=(dx, None)))
    tdk = med(lambda: rs.conv_bwd(x, kk, dy, need_dx=False, out=(None, dk)))
    ta = med(lambda: rs.conv_bwd(x, kk, dy, algo="scatter_atomic", need_dk=False, out=(dx, None)), reps=5)
    flops = 2.0 * N * H * W * C * C * k * k
    fp = fp32_peak_tflops()
    out["f1_conv_16x16x256x256_k3"] = {
        "fwd_us": round(tf * 1e6, 1), "bwd_us": round(tg * 1e6, 1),
        "bwd_dx_gather_us": round(tdx * 1e6, 1), "bwd_dx_atomic_us": round(ta * 1e6, 1),
        "bwd_dk_us": round(tdk * 1e6, 1), "atomic_over_gather": round(ta / tdx, 2),
        "paper_atomic_over_gather": round(68.0 / 6.0, 2),
        "roofline": {"bound": "alu", "unit": "TFLOP/s", "peak": round(fp, 1),
                     "peak_source": "148 SMs x 128 FP32 FMA/clk x 2 x sm_max_mhz (B200_PROFILING.md unit counts)",
                     "fwd_frac": round(flops / tf / 1e12 / fp, 3), "dx_gather_frac": round(flops / tdx / 1e12 / fp, 3),
                     "dk_frac": round(flops / tdk / 1e12 / fp, 3)},
    }
    del x, dy, y, dx
    # f4: the checkpointing study, 2560 x 1600, kernels 1 x 5 and 3 x 5;
    # the paper's CPU times (ms: inline / root / compute_at) are context only
    paper_ms = {(1, 5): (5.6, 10.1, 9.7), (3, 5): (66.2, 18.7, 12.3)}
    H, W = 1600, 2560
    inp = torch.rand(1, H, W, device=dev, generator=g)
    tgt = torch.rand(1, H, W, device=dev, generator=g)
    d = torch.empty_like(inp)
    for kh, kw in ((1, 5), (3, 5)):
        kk = torch.randn(kh, kw) / (kh * kw) ** 0.5
        r = {}
        for sch in ("inline", "root", "at"):
            t = med(lambda: rs.convloss_grad(inp, kk, tgt, schedule=sch, out=d))  # noqa: B023
            r[f"{sch}_us"] = round(t * 1e6, 1)
            # compulsory bytes: in + target read, d_in written (root adds R write + read)
            r[f"{sch}_hbm_frac"] = round(12.0 * H * W / t / 1e9 / peak, 3)
        r["paper_cpu_ms_inline_root_at"] = paper_ms[(kh, kw)]
        out[f"f4_convloss_2560x1600_k{kh}x{kw}"] = r
    xu = torch.randn(1, 3, 400, 640, device=dev, generator=g)
    yu = torch.empty(1, 3, 1600, 2560, device=dev)
    dxu = torch.empty_like(xu)
    tu_f = med(lambda: rs.upsample4_fwd(xu, out=yu))
    tu_b = med(lambda: rs.upsample4_bwd(yu, out=dxu))
    bu = 4.0 * xu.numel() * 17  # 1 + 16 floats per input element
    out["f4_upsample4_1x3x400x640"] = {"fwd_us": round(tu_f * 1e6, 1), "bwd_us": round(tu_b * 1e6, 1),
                                       "fwd_hbm_frac": round(bu / tu_f / 1e9 / peak, 3),
                                       "bwd_hbm_frac": round(bu / tu_b / 1e9 / peak, 3)}
    # f3: bicubic STN at the paper's STN shape (4 x 16 x 512^2) and a volumetric STN
    import synth
    si = synth.stn_inputs(4, 16, 512, 512, cfg=2, device=dev)
    yb, dxb, dtb = torch.empty_like(si["dy"]), torch.empty_like(si["x"]), torch.empty_like(si["theta"])
    tbf = med(lambda: rs.stn_bicubic_fwd(si["x"], si["theta"], out=yb))
    tbb = med(lambda: rs.stn_bicubic_bwd(si["x"], si["theta"], si["dy"], out=(dxb, dtb)))
    P = 4 * 512 * 512
    out["f3_stn_bicubic_4x16x512x512"] = {
        "fwd_us": round(tbf * 1e6, 1), "bwd_us": round(tbb * 1e6, 1),
        "fwd_bwd_mpix_s": round(P / (tbf + tbb) / 1e6, 1),
        "fwd_roofline_frac": round(BYTES[("stn", "fwd")](16) * P / tbf / 1e9 / peak, 3),
        "bwd_roofline_frac": round(BYTES[("stn", "bwd")](16) * P / tbb / 1e9 / peak, 3)}
    tlf = med(lambda: rs.stn_lanczos_fwd(si["x"], si["theta"], out=yb))
    tlb = med(lambda: rs.stn_lanczos_bwd(si["x"], si["theta"], si["dy"], out=(dxb, dtb)))
    out["f3_stn_lanczos3_4x16x512x512"] = {
        "fwd_us": round(tlf * 1e6, 1), "bwd_us": round(tlb * 1e6, 1),
        "fwd_bwd_mpix_s": round(P / (tlf + tlb) / 1e6, 1),
        "fwd_roofline_frac": round(BYTES[("stn", "fwd")](16) * P / tlf / 1e9 / peak, 3),
        "bwd_roofline_frac": round(BYTES[("stn", "bwd")](16) * P / tlb / 1e9 / peak, 3)}
    del si, yb, dxb
    x3 = torch.randn(2, 4, 96, 96, 96, device=dev, generator=g)
    d3 = torch.randn(2, 4, 96, 96, 96, device=dev, generator=g)
    th3 = torch.eye(3, 4, device=dev).expand(2, 3, 4).contiguous() + 0.05 * torch.randn(2, 3, 4, device=dev, generator=g)
    y3, dx3, dt3 = torch.empty_like(x3), torch.empty_like(x3), torch.empty_like(th3)
    t3f = med(lambda: rs.stn3d_fwd(x3, th3, out=y3))
    t3b = med(lambda: rs.stn3d_bwd(x3, th3, d3, out=(dx3, dt3)))
    P3 = 2 * 96 ** 3
    out["f3_stn3d_2x4x96^3"] = {
        "fwd_us": round(t3f * 1e6, 1), "bwd_us": round(t3b * 1e6, 1),
        "fwd_bwd_mvox_s": round(P3 / (t3f + t3b) / 1e6, 1),
        "fwd_roofline_frac": round(8.0 * 4 * P3 / t3f / 1e9 / peak, 3),
        "bwd_roofline_frac": round(12.0 * 4 * P3 / t3b / 1e9 / peak, 3)}
    del fl
    return {"l2": "flushed (256 MB write) before every call; median of 10", "rows": out}


# --------------------------------------------------------------------------- cpu baseline
def cpu_baseline(s, w, b, budget_s=12.0):
    """The fp64 oracle as it stands on sample 0 of each layer, repeated while under budget."""
    import oracle

    sub = lambda d: {k: v[:1].double().cpu().numpy() for k, v in d.items()}  # noqa: E731
    S, Wp, B = sub(s), sub(w), sub(b)
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.stn_fwd(S["x"], S["theta"])
        oracle.stn_bwd(S["x"], S["theta"], S["dy"])
        oracle.warp_fwd(Wp["x"], Wp["flow"])
        oracle.warp_bwd(Wp["x"], Wp["flow"], Wp["dy"])
        oracle.bslice_fwd(B["grid"], B["guide"], B["x"])
        oracle.bslice_bwd(B["grid"], B["guide"], B["x"], B["dy"])
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": round(reps * H * W / dt / 1e6, 4), "unit": UNIT, "cores": oracle.get_threads(),
            "kind": "oracle",
            "sample": f"{reps} x one sample (1 x 1024^2) of each layer of the step (STN C=16, warp C=3, "
                      f"bslice 16x16x8), fp64 C oracle, OpenMP; host os.cpu_count()={os.cpu_count()}"}


def cpu_configs(budget_1t_s=20.0):
    """the oracle (fp64 fwd + naive scatter adjoint) on the full
    configs[0..3] (K1 STN 1x3x16^2, K2 STN 4x16x512^2, K3 warp 8x3x384x512, K4 bslice
    4x1024^2 16x16x8), once with all host threads and once with 1 thread (the 1-thread
    run stops after the budget; configs not reached are reported as skipped)."""
    import oracle
    import synth

    cases = [
        ("K1_stn_1x3x16x16", 1 * 16 * 16, lambda: synth.stn_inputs(1, 3, 16, 16, cfg=1), "stn"),
        ("K2_stn_4x16x512x512", 4 * 512 * 512, lambda: synth.stn_inputs(4, 16, 512, 512, cfg=2), "stn"),
        ("K3_warp_8x3x384x512", 8 * 384 * 512, lambda: synth.warp_inputs(8, 3, 384, 512, cfg=3), "warp"),
        ("K4_bslice_4x1024x1024_g16x16x8", 4 * 1024 * 1024,
         lambda: synth.bslice_inputs(4, 1024, 1024, 8, 16, 16, cfg=4), "bslice"),
    ]

    def run(layer, d):
        if layer == "stn":
            oracle.stn_fwd(d["x"], d["theta"])
            oracle.stn_bwd(d["x"], d["theta"], d["dy"])
        elif layer == "warp":
            oracle.warp_fwd(d["x"], d["flow"])
            oracle.warp_bwd(d["x"], d["flow"], d["dy"])
        else:
            oracle.bslice_fwd(d["grid"], d["guide"], d["x"])
            oracle.bslice_bwd(d["grid"], d["guide"], d["x"], d["dy"])

    nthr = oracle.get_threads()
    out = {"threads_all": nthr, "host_cpu_count": os.cpu_count(), "cases": {}}
    spent_1t = 0.0
    for name, P, make, layer in cases:
        d = {k: v.double().numpy() for k, v in make().items()}
        t0 = time.perf_counter()
        run(layer, d)
        ta = time.perf_counter() - t0
        r = {"fwd_bwd_s_all_threads": round(ta, 4), "mpix_s_all_threads": round(P / ta / 1e6, 3)}
        if spent_1t < budget_1t_s:
            oracle.set_threads(1)
            try:
                t0 = time.perf_counter()
                run(layer, d)
                t1 = time.perf_counter() - t0
            finally:
                oracle.set_threads(nthr)
            spent_1t += t1
            r.update({"fwd_bwd_s_1_thread": round(t1, 4), "mpix_s_1_thread": round(P / t1 / 1e6, 3)})
        else:
            r["1_thread"] = "skipped (1-thread budget spent)"
        out["cases"][name] = r
    return out


# --------------------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    import synth

    s = synth.stn_inputs(1, C_STN, H, W, cfg=5)
    w = synth.warp_inputs(1, C_WARP, H, W, cfg=5)
    b = synth.bslice_inputs(1, H, W, D, GH, GW, cfg=5)
    S = {k: v.double().numpy() for k, v in s.items()}
    Wp = {k: v.double().numpy() for k, v in w.items()}
    B = {k: v.double().numpy() for k, v in b.items()}

    def step():
        oracle.stn_fwd(S["x"], S["theta"])
        oracle.stn_bwd(S["x"], S["theta"], S["dy"])
        oracle.warp_fwd(Wp["x"], Wp["flow"])
        oracle.warp_bwd(Wp["x"], Wp["flow"], Wp["dy"])
        oracle.bslice_fwd(B["grid"], B["guide"], B["x"])
        oracle.bslice_bwd(B["grid"], B["guide"], B["x"], B["dy"])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = round(H * W / dt / 1e6, 4)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/, seeded)",
        "config": config_dict(1),
        "cpu_baseline": {"value": v, "unit": UNIT, "kind": "oracle", "cores": oracle.get_threads(),
                         "sample": "each step = one 1024^2 sample (of the 64) of each layer, fp64 C "
                                   "oracle, OpenMP; value = that sample's pixels / step time"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- main
class DeviceClock:
    """Per-step device timing on the launching stream (CUDA events)."""

    def __init__(self, steps, ncalls, stream):
        self.stream = stream
        self.ev = [[torch.cuda.Event(enable_timing=True) for _ in range(ncalls + 1)] for _ in range(steps)]

    def mark(self, k, i):
        self.ev[k][i].record(self.stream)

    def finish(self):
        torch.cuda.synchronize()

    def seconds(self, k, i, j):
        return self.ev[k][i].elapsed_time(self.ev[k][j]) * 1e-3


class HostClock:
    """--dry-run (CPU plumbing only): wall-clock marks."""

    def __init__(self, steps, ncalls, stream=None):
        self.t = [[0.0] * (ncalls + 1) for _ in range(steps)]

    def mark(self, k, i):
        self.t[k][i] = time.perf_counter()

    def finish(self):
        pass

    def seconds(self, k, i, j):
        return self.t[k][j] - self.t[k][i]


def dry_calls(nb):
    """--dry-run stand-in for the six calls: a little CPU work per call, no product code."""
    a = torch.ones(nb, 256, 256)
    return [(n, (lambda: a.mul_(1.0))) for n in
            ("stn_fwd", "stn_bwd", "warp_fwd", "warp_bwd", "bslice_fwd", "bslice_bwd")]


def timed_steps(calls, steps, world, clock):
    """K timed steps.  Every step: events around each of the six calls on the launching
    stream; between steps a barrier (outside the events).  Per step and per call the
    MAX over ranks, then the median over steps; also the max-over-ranks
    total of the K steps (the bracketed-region number)."""
    barrier(world)
    for k in range(steps):
        clock.mark(k, 0)
        for ci, (_, fn) in enumerate(calls):
            fn()
            clock.mark(k, ci + 1)
        if world > 1:
            clock.finish()
            barrier(world)
    clock.finish()
    nc = len(calls)
    per = [[clock.seconds(k, ci, ci + 1) for ci in range(nc)] for k in range(steps)]
    tot = [clock.seconds(k, 0, nc) for k in range(steps)]
    flat = max_over_ranks(world, tot + [v for row in per for v in row])
    tot_max, per_max = flat[:steps], flat[steps:]
    per_max = [per_max[k * nc:(k + 1) * nc] for k in range(steps)]
    step_med = statistics.median(tot_max)
    call_med = [statistics.median(per_max[k][ci] for k in range(steps)) for ci in range(nc)]
    return step_med, call_med, sum(tot_max)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-paper-shapes", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-next", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU plumbing test of the rank loop (gloo, stand-in calls, no product code)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    spawn_ranks(args)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    n0, nb = shard(world, rank)
    if args.dry_run:
        calls, clock_t, rs = dry_calls(nb), HostClock, None
        stream = None
    else:
        from paper_1904_12228_b200 import rsgrad as rs

        dev = torch.device("cuda", local if world > 1 else 0)
        s, w, b = make_inputs(n0, nb, dev)
        o = alloc_outputs(s, w, b)
        calls = step_calls(rs, s, w, b, o)
        stream = torch.cuda.current_stream()
        clock_t = DeviceClock
    for _ in range(args.warmup):
        for _, fn in calls:
            fn()
    if not args.dry_run:
        torch.cuda.synchronize()

    # ---- timed region
    clock = clock_t(args.steps, len(calls), stream)
    clocks = ClockSampler(torch.cuda.current_device()) if (rank == 0 and not args.dry_run) else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    if rs is not None:
        rs.launch_count(reset=True)
    t_step, per_call, total_s = timed_steps(calls, args.steps, world, clock)
    launches = rs.launch_count() if rs is not None else 0
    barrier(world)
    clk = clocks.stop() if clocks else None
    P_global = BATCH * H * W
    value = P_global / t_step / 1e6

    # ---- e2e: the same step through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e and not args.dry_run:
        e2e = run_e2e(rs, s, w, b, args, world)

    if rank != 0:
        return
    peak, peak_src = peak_hbm()
    names = [n for n, _ in calls]
    P_rank = nb * H * W
    layers = {}
    for L in ("stn", "warp", "bslice"):
        tf, tb = per_call[names.index(f"{L}_fwd")], per_call[names.index(f"{L}_bwd")]
        C = {"stn": C_STN, "warp": C_WARP, "bslice": 3}[L]
        layers[L] = {
            "fwd_bwd_mpix_s": round(P_global / (tf + tb) / 1e6, 1),
            "fwd_ms": round(tf * 1e3, 4), "bwd_ms": round(tb * 1e3, 4),
            "fwd_roofline_frac": round(BYTES[(L, "fwd")](C) * P_rank / tf / 1e9 / peak, 3),
            "bwd_roofline_frac": round(BYTES[(L, "bwd")](C) * P_rank / tb / 1e9 / peak, 3),
        }
    dom = max(range(len(calls)), key=lambda i: per_call[i])
    dname = names[dom]
    achieved = CALL_BYTES[dname] * P_rank / per_call[dom] / 1e9
    roof = {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": ncu_traffic(dname, P_rank),
            "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write per pixel x pixels per launch)",
            "algorithmic_bytes_per_launch": CALL_BYTES[dname] * P_rank, "peak_source": peak_src}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (synth/: seeded per-sample recipe, generated on device)",
        "config": config_dict(world),
        "timing": {"ms_per_step": "median over the K steps of the per-step max over ranks (CUDA events on the "
                                  "launching stream; a barrier between steps, outside the events)",
                   "total_ms_k_steps_max_over_ranks": round(total_s * 1e3, 4)},
        "layers": layers, "roofline": roof, "gpu_launches": launches,
        "clocks": clk, "e2e": e2e,
    }
    if args.dry_run:
        line["dry_run"] = True
        line["data"] = "none (--dry-run: CPU stand-in calls, plumbing only)"
        line["per_rank_shards"] = [list(shard(world, r)) for r in range(world)]
    if world == 1 and not args.no_cpu and not args.dry_run:
        line["cpu_baseline"] = cpu_baseline(s, w, b)
        line["cpu_baseline"]["configs"] = cpu_configs()
    if world == 1 and not args.no_paper_shapes and not args.dry_run:
        line["paper_shapes"] = paper_shapes(rs, peak)
    if world == 1 and not args.no_next and not args.dry_run:
        line["next_rows"] = next_rows(rs, peak)
    print(json.dumps(line), flush=True)


def ncu_traffic(call, P_rank):
    """dram_bytes_read + dram_bytes_write per launch of `call`, from the committed
    `ncu --set full` capture (profiles/ncu_traffic.json, measured per pixel at a
    smaller batch and scaled to this launch's pixels), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(call)
        if v is None:
            return None
        return round(v["per_pixel"] * P_rank)
    except Exception:  # noqa: BLE001
        return None


def run_e2e(rs, s, w, b, args, world):
    """Host-buffer step: the library copies every input H2D and output D2H on the stream."""
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 0
    nb_full = s["x"].shape[0]
    per_sample = sum(v[0].numel() * 4 for d in (s, w, b) for v in d.values()) * 2
    nb = nb_full
    while nb > 1 and nb * per_sample * 1.5 > avail:
        nb //= 2
    pick = lambda d: {k: v[:nb].cpu().pin_memory() for k, v in d.items()}  # noqa: E731
    hs, hw, hb = pick(s), pick(w), pick(b)
    ho = alloc_outputs(hs, hw, hb, host=True)
    calls = step_calls(rs, hs, hw, hb, ho, sync=False)  # one stream sync per step (below)
    h2d = (sum(hs[k].numel() for k in ("x", "theta")) + sum(hs[k].numel() for k in ("x", "theta", "dy"))
           + sum(hw[k].numel() for k in ("x", "flow")) + sum(hw[k].numel() for k in ("x", "flow", "dy"))
           + sum(hb[k].numel() for k in ("grid", "guide", "x"))
           + sum(hb[k].numel() for k in ("grid", "guide", "x", "dy"))) * 4
    d2h = sum(v.numel() for k, v in ho.items() if not k.startswith("_")) * 4
    # a caller-owned staging buffer (3 streams x the largest chunk's host tensors +
    # workspace: the library carves its per-chunk buffers from it, no per-call allocation)
    stage = torch.empty(int(1.5 * 2**30), dtype=torch.uint8, device=s["x"].device)
    rs.set_host_staging(stage)
    for _, fn in calls:  # warm-up
        fn()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        for _, fn in calls:
            fn()
        torch.cuda.current_stream().synchronize()  # the step's results are readable on the host
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    rs.set_host_staging(None)
    del stage
    dt = max(e0.elapsed_time(e1) * 1e-3 / steps, 1e-9)
    dt = max_over_ranks(world, [max(dt, wall)])[0]
    v = world * nb * H * W / dt / 1e6
    return {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "samples_per_rank": nb, "steps": steps,
            "note": "pinned host buffers passed as host pointers to the C ABI: the library stages "
                    "them in up to 32 sample chunks on three internal streams (H2D / kernels / D2H overlap; "
                    "staging carved from a caller-owned 1.5 GB device buffer, rsgrad_set_host_staging); "
                    "one stream sync per step; wall clock, max over ranks"}


if __name__ == "__main__":
    main()
