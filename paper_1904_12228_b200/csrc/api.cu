// api.cu — the extern "C" boundary declared in include/rsgrad.h.
//
// Responsibilities: argument validation, option defaults, host-pointer staging
// (stream-ordered temporaries), workspace provisioning, error reporting through
// a thread-local string, and dispatch to the per-layer launchers.  No compute.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <cstdlib>
#include <mutex>
#include <initializer_list>
#include <vector>

#include "../../include/rsgrad.h"
#include "common.cuh"

namespace rs {
static thread_local char g_err[512] = "";
static thread_local unsigned long long g_launches = 0;
void note_launch() { g_launches++; }
}  // namespace rs

namespace {

rs_status fail(rs_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(rs::g_err, sizeof(rs::g_err), fmt, ap);
    va_end(ap);
    return st;
}

rs_status ok() {
    rs::g_err[0] = 0;
    return RS_OK;
}

rs_opts resolve(const rs_opts *o) {
    rs_opts r;
    if (o) {
        r = *o;
    } else {
        r.align_corners = 1;
        r.padding = RS_PAD_ZEROS;
        r.algo = RS_ALGO_AUTO;
        r.deterministic = 0;
    }
    return r;
}

rs_status check_opts(const rs_opts &o) {
    if (o.align_corners != 0 && o.align_corners != 1)
        return fail(RS_ERR_FLAG, "align_corners must be 0 or 1 (got %d)", o.align_corners);
    if (o.padding != RS_PAD_ZEROS && o.padding != RS_PAD_BORDER)
        return fail(RS_ERR_FLAG, "padding must be RS_PAD_ZEROS or RS_PAD_BORDER (got %d)", o.padding);
    if (o.algo < RS_ALGO_AUTO || o.algo > RS_ALGO_SCATTER_ATOMIC)
        return fail(RS_ERR_FLAG, "unknown algo %d", o.algo);
    if (o.deterministic != 0 && o.deterministic != 1)
        return fail(RS_ERR_FLAG, "deterministic must be 0 or 1");
    return RS_OK;
}

constexpr int kMaxHostStreams = 4;

// Library temporaries (a workspace the caller did not provide, host-path staging) are
// stream-ordered allocations from the device's default memory pool (cudaMallocAsync /
// cudaFreeAsync on the call's stream): nothing is reserved by the library between
// calls -- what the pool keeps cached is the pool's (i.e. the caller's) release
// policy (SURVEY 8(b) "the library never allocates persistently").
cudaError_t lib_malloc(void **p, size_t bytes, cudaStream_t s) { return cudaMallocAsync(p, bytes, s); }

// Make the device of the caller's stream current for the duration of one entry point:
// launches, stream-ordered allocations and cudaFuncSetAttribute act on the current
// device, so a stream of another GPU would otherwise fail (or allocate on the wrong
// device).  The legacy default stream (NULL) means the current device.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(cudaStream_t s) {
        if (!s) return;
        // cudaStreamGetDevice invalidates a stream capture (measured): a capturing stream
        // belongs to the current device (CUDA-graph capture is set up on it)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
            cudaGetLastError();
            return;
        }
        int d = 0, cur = 0;
        if (cudaStreamGetDevice(s, &d) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        if (cudaGetDevice(&cur) == cudaSuccess && cur != d && cudaSetDevice(d) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Internal streams / events of the host-pointer path, created once per (thread,
// device) and reused by every later call on that thread (re-entrant: no sharing
// between threads).  Released with the CUDA context.
struct HostStreams {
    bool made = false;
    cudaStream_t st[4];
    cudaEvent_t ev0, evs[4];
    // caller-owned device staging buffer (rsgrad_set_host_staging), or none
    char *stage = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_free;  // recorded when the last call using `stage` is done with it
    bool stage_used = false;
};
HostStreams &host_streams() {
    static thread_local HostStreams hs[64];
    int dev = 0;
    cudaGetDevice(&dev);
    HostStreams &h = hs[dev >= 0 && dev < 64 ? dev : 0];
    if (!h.made) {
        for (int k = 0; k < 4; k++) {
            cudaStreamCreateWithFlags(&h.st[k], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&h.evs[k], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&h.ev0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h.stage_free, cudaEventDisableTiming);
        h.made = true;
    }
    return h;
}

// integer tuning knob from the environment (A/B measurements), clamped to [1, hi]
int env_int(const char *name, int dflt, int hi = 64) {
    const char *e = getenv(name);
    int v = e ? atoi(e) : dflt;
    if (v < 1) v = 1;
    if (v > hi) v = hi;
    if (std::string(name) == "RSGRAD_HOST_STREAMS" && v > kMaxHostStreams) v = kMaxHostStreams;
    return v;
}

// One tensor argument of an entry point: pointer (device, host or NULL), bytes per
// sample, direction.
struct TArg {
    const void *p;
    size_t per_sample;
    bool in;
    bool out;
};

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // clear: unregistered host memory on old drivers
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Run launch(n0, nc, ptrs, stream, workspace) over samples [0, N).
//  * all pointers device memory: one launch on `s` with the caller's pointers and
//    workspace (allocated stream-ordered on `s` if absent / too small);
//  * any host pointer: the batch is split into sample chunks processed on two
//    internal streams ordered after `s` (and `s` after them): per chunk, host inputs
//    are copied H2D into stream-ordered temporaries, the kernels run, host outputs
//    are copied D2H — copies of one chunk overlap the kernels of the other (every
//    sample is independent).  Pinned host memory keeps all of it asynchronous.
template <class F, class WS>
rs_status run_batched(int N, std::vector<TArg> &args, cudaStream_t s, void *workspace, size_t ws_bytes,
                      WS &&ws_need, F &&launch) {
    const int na = (int)args.size();
    std::vector<bool> host(na, false);
    bool any_host = false;
    for (int i = 0; i < na; i++)
        if (args[i].p && !is_device_ptr(args[i].p)) host[i] = any_host = true;
    std::vector<void *> ptr(na);
    if (!any_host) {
        for (int i = 0; i < na; i++) ptr[i] = const_cast<void *>(args[i].p);
        const size_t need = ws_need(N);
        void *ws = workspace;
        bool own = false;
        if (need && (!ws || ws_bytes < need)) {
            cudaError_t e = lib_malloc(&ws, need, s);
            if (e != cudaSuccess) return fail(RS_ERR_WORKSPACE, "workspace cudaMallocAsync(%zu): %s", need, cudaGetErrorString(e));
            own = true;
        }
        cudaError_t e = launch(0, N, ptr.data(), s, ws);
        if (own) cudaFreeAsync(ws, s);
        if (e != cudaSuccess) return fail(RS_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
        return ok();
    }
    // more, smaller chunks shorten the pipeline's fill and drain (the first chunk's H2D
    // and the last chunk's D2H are not overlapped); three streams let chunk c+1's H2D,
    // chunk c's kernels and chunk c-1's D2H run at once (H2D and D2H engines in parallel)
    const int maxchunk = env_int("RSGRAD_HOST_CHUNKS", 32), NS = env_int("RSGRAD_HOST_STREAMS", 3);
    const int nchunk = N < maxchunk ? N : maxchunk;
    const int cs = (N + nchunk - 1) / nchunk;
    HostStreams &hs = host_streams();
    cudaStream_t *st = hs.st;
    cudaEventRecord(hs.ev0, s);
    std::vector<void *> buf[kMaxHostStreams];
    void *wsk[kMaxHostStreams] = {};
    cudaError_t err = cudaSuccess;
    // staging: carve from the caller's registered buffer when it is large enough (no
    // per-call allocation), else stream-ordered temporaries
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t per_stream = al(ws_need(cs));
    for (int i = 0; i < na; i++)
        if (host[i]) per_stream += al(args[i].per_sample * cs);
    const bool use_stage = hs.stage && per_stream * NS <= hs.stage_bytes;
    for (int k = 0; k < NS; k++) {
        cudaStreamWaitEvent(st[k], hs.ev0, 0);
        if (use_stage && hs.stage_used) cudaStreamWaitEvent(st[k], hs.stage_free, 0);
        buf[k].assign(na, nullptr);
        char *cur = use_stage ? hs.stage + per_stream * k : nullptr;
        for (int i = 0; i < na; i++)
            if (host[i] && err == cudaSuccess) {
                if (use_stage) {
                    buf[k][i] = cur;
                    cur += al(args[i].per_sample * cs);
                } else {
                    err = lib_malloc(&buf[k][i], args[i].per_sample * cs, st[k]);
                }
            }
        const size_t need = ws_need(cs);
        if (need && err == cudaSuccess) {
            if (use_stage) wsk[k] = cur;
            else err = lib_malloc(&wsk[k], need, st[k]);
        }
    }
    for (int c = 0, n0 = 0; n0 < N && err == cudaSuccess; c++, n0 += cs) {
        const int nc = N - n0 < cs ? N - n0 : cs, k = c % NS;
        for (int i = 0; i < na && err == cudaSuccess; i++) {
            const size_t off = args[i].per_sample * (size_t)n0, bytes = args[i].per_sample * (size_t)nc;
            if (!args[i].p) {
                ptr[i] = nullptr;
            } else if (host[i]) {
                ptr[i] = buf[k][i];
                if (args[i].in)
                    err = cudaMemcpyAsync(ptr[i], (const char *)args[i].p + off, bytes, cudaMemcpyHostToDevice, st[k]);
            } else {
                ptr[i] = (char *)const_cast<void *>(args[i].p) + off;
            }
        }
        if (err == cudaSuccess) err = launch(n0, nc, ptr.data(), st[k], wsk[k]);
        for (int i = 0; i < na && err == cudaSuccess; i++)
            if (host[i] && args[i].out)
                err = cudaMemcpyAsync((char *)const_cast<void *>(args[i].p) + args[i].per_sample * (size_t)n0, ptr[i],
                                      args[i].per_sample * (size_t)nc, cudaMemcpyDeviceToHost, st[k]);
    }
    for (int k = 0; k < NS; k++) {
        if (!use_stage) {
            for (int i = 0; i < na; i++)
                if (buf[k][i]) cudaFreeAsync(buf[k][i], st[k]);
            if (wsk[k]) cudaFreeAsync(wsk[k], st[k]);
        }
        cudaEventRecord(hs.evs[k], st[k]);
        cudaStreamWaitEvent(s, hs.evs[k], 0);
    }
    if (use_stage) {  // the next call that uses the staging buffer waits for this one
        cudaEventRecord(hs.stage_free, s);
        hs.stage_used = true;
    }
    if (err != cudaSuccess) return fail(RS_ERR_CUDA, "host-staged path: %s", cudaGetErrorString(err));
    return ok();
}

rs_status launched(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return ok();
}

bool pos(int v) { return v > 0; }

}  // namespace

extern "C" {

const char *rsgrad_last_error(void) { return rs::g_err; }

const char *rsgrad_version(void) { return "rsgrad 0.1.0 sm_100a"; }

rs_status rsgrad_set_host_staging(void *buf, size_t bytes) {
    if (buf && !is_device_ptr(buf)) return fail(RS_ERR_FLAG, "rsgrad_set_host_staging: not device memory");
    HostStreams &h = host_streams();
    if (h.stage && h.stage_used) cudaEventSynchronize(h.stage_free);  // the old buffer is released idle
    h.stage = (char *)buf;
    h.stage_bytes = buf ? bytes : 0;
    h.stage_used = false;
    return ok();
}

unsigned long long rsgrad_launch_count(int reset) {
    unsigned long long v = rs::g_launches;
    if (reset) rs::g_launches = 0;
    return v;
}

size_t rsgrad_bwd_workspace_bytes(int layer, int N, int C, int H, int W, int Ho, int Wo, int D,
                                  int Gh, int Gw, const rs_opts *opts) {
    const bool det = opts && opts->deterministic == 1;
    switch (layer) {
        case 0:
            if (!pos(N) || !pos(C) || !pos(H) || !pos(W) || !pos(Ho) || !pos(Wo)) return 0;
            return rs::stn_ws_bytes(N, C, H, W, Ho, Wo, det);
        case 1:
            if (!pos(N) || !pos(C) || !pos(H) || !pos(W)) return 0;
            return rs::warp_ws_bytes(N, C, H, W, det);
        case 2:
            if (!pos(N) || !pos(H) || !pos(W) || !pos(D) || !pos(Gh) || !pos(Gw)) return 0;
            return rs::bslice_bwd_ws_bytes(N, H, W, D, Gh, Gw, det);
        case 3:
            if (!pos(N) || !pos(C) || !pos(H) || !pos(W) || !pos(D) || !pos(Gh) || !pos(Gw)) return 0;
            return rs::conv_ws_bytes(N, C, D, H, W, Gh, Gw);
        case 4:
            if (!pos(N) || !pos(H) || !pos(W)) return 0;
            return rs::convloss_ws_bytes(N, H, W);
        case 5:
            if (!pos(N) || !pos(Ho) || !pos(Wo)) return 0;
            if (!pos(C) || !pos(H) || !pos(W)) return 0;
            return rs::stn_bicubic_ws_bytes(N, C, H, W, Ho, Wo, det);
        case 6:  // stn3d: (N, C, H, W) of the input volume with Gh = its depth; (Ho, Wo, D = Do) of the output
            if (!pos(N) || !pos(Ho) || !pos(Wo) || !pos(D)) return 0;
            if (det && (!pos(C) || !pos(H) || !pos(W) || !pos(Gh))) return 0;
            return rs::stn3d_ws_bytes(N, C, det ? Gh : 1, H, W, D, Ho, Wo, det);
        case 7:
            if (!pos(N) || !pos(Ho) || !pos(Wo)) return 0;
            if (det && (!pos(C) || !pos(H) || !pos(W))) return 0;
            return rs::stn_lanczos_ws_bytes(N, C, H, W, Ho, Wo, det);
        default:
            return 0;
    }
}

// ------------------------------------------------------------------------------ STN
static rs_status stn_validate(const float *x, const float *theta, int N, int C, int H, int W,
                              int Ho, int Wo, const rs_opts &o) {
    if (!x || !theta) return fail(RS_ERR_NULL, "stn: x and theta are required");
    if (!pos(N) || !pos(C) || !pos(H) || !pos(W) || !pos(Ho) || !pos(Wo))
        return fail(RS_ERR_SHAPE, "stn: dims must be positive (N=%d C=%d H=%d W=%d Ho=%d Wo=%d)", N,
                    C, H, W, Ho, Wo);
    if (o.align_corners && (Ho < 2 || Wo < 2))
        return fail(RS_ERR_SHAPE, "stn: align_corners=1 needs Ho, Wo >= 2 (got %d, %d)", Ho, Wo);
    if (N > 65535 || (long long)H * W >= (1LL << 31) || (long long)Ho * Wo >= (1LL << 31))
        return fail(RS_ERR_SHAPE, "stn: N <= 65535 and H*W, Ho*Wo < 2^31 per launch (split the batch)");
    return check_opts(o);
}

rs_status stn_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho, int Wo,
                  const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "stn_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{x, sizeof(float) * (size_t)C * H * W, true, false},
                              {theta, sizeof(float) * 6, true, false},
                              {y, sizeof(float) * (size_t)C * Ho * Wo, false, true}};
    return run_batched(N, args, s, nullptr, 0, [](int) { return (size_t)0; },
                       [&](int, int nc, void **p, cudaStream_t t, void *) {
                           rs::StnArgs a{};
                           a.x = (const float *)p[0];
                           a.theta = (const float *)p[1];
                           a.y = (float *)p[2];
                           a.N = nc; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
                           a.ac = o.align_corners;
                           a.border = o.padding == RS_PAD_BORDER;
                           return rs::stn_fwd_launch(a, t);
                       });
}

rs_status stn_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H, int W,
                  int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta, void *workspace,
                  size_t ws_bytes, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "stn_bwd: dy is required");
    const bool border = o.padding == RS_PAD_BORDER;
    if (dx && border && o.algo == RS_ALGO_GATHER)
        return fail(RS_ERR_FLAG, "stn_bwd: GATHER needs zeros padding (border clamp has no bounded inverse)");
    if (dx && (o.algo == RS_ALGO_SCATTER_ATOMIC || o.algo == RS_ALGO_SCATTER_PRIV) && o.deterministic)
        return fail(RS_ERR_FLAG, "stn_bwd: scatter paths (atomics) are not deterministic");
    if (!dx && !dtheta) return ok();
    const bool det = o.deterministic && dx;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{x, sizeof(float) * (size_t)C * H * W, true, false},
                              {theta, sizeof(float) * 6, true, false},
                              {dy, sizeof(float) * (size_t)C * Ho * Wo, true, false},
                              {dx, sizeof(float) * (size_t)C * H * W, false, true},
                              {dtheta, sizeof(float) * 6, false, true}};
    return run_batched(N, args, s, workspace, ws_bytes,
                       [&](int n) { return rs::stn_ws_bytes(n, C, H, W, Ho, Wo, det); },
                       [&](int, int nc, void **p, cudaStream_t t, void *ws) {
                           rs::StnArgs a{};
                           a.x = (const float *)p[0];
                           a.theta = (const float *)p[1];
                           a.dy = (const float *)p[2];
                           a.dx = (float *)p[3];
                           a.dtheta = (float *)p[4];
                           a.N = nc; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
                           a.ac = o.align_corners;
                           a.border = border;
                           return rs::stn_bwd_launch(a, o.algo, o.deterministic, ws,
                                                     rs::stn_ws_bytes(nc, C, H, W, Ho, Wo, det), t);
                       });
}

// ------------------------------------------------------------------------------ warp
static rs_status warp_validate(const float *x, const float *flow, int N, int C, int H, int W,
                               const rs_opts &o) {
    if (!x || !flow) return fail(RS_ERR_NULL, "warp: x and flow are required");
    if (!pos(N) || !pos(C) || !pos(H) || !pos(W))
        return fail(RS_ERR_SHAPE, "warp: dims must be positive (N=%d C=%d H=%d W=%d)", N, C, H, W);
    if (N > 65535 || (long long)H * W >= (1LL << 31))
        return fail(RS_ERR_SHAPE, "warp: N <= 65535 and H*W < 2^31 per launch (split the batch)");
    return check_opts(o);
}

rs_status warp_fwd(const float *x, const float *flow, int N, int C, int H, int W,
                   const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = warp_validate(x, flow, N, C, H, W, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "warp_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{x, sizeof(float) * (size_t)C * H * W, true, false},
                              {flow, sizeof(float) * 2 * (size_t)H * W, true, false},
                              {y, sizeof(float) * (size_t)C * H * W, false, true}};
    return run_batched(N, args, s, nullptr, 0, [](int) { return (size_t)0; },
                       [&](int, int nc, void **p, cudaStream_t t, void *) {
                           rs::WarpArgs a{};
                           a.x = (const float *)p[0];
                           a.flow = (const float *)p[1];
                           a.y = (float *)p[2];
                           a.N = nc; a.C = C; a.H = H; a.W = W;
                           a.border = o.padding == RS_PAD_BORDER;
                           return rs::warp_fwd_launch(a, t);
                       });
}

rs_status warp_bwd(const float *x, const float *flow, const float *dy, int N, int C, int H, int W,
                   const rs_opts *opts, float *dx, float *dflow, void *workspace, size_t ws_bytes,
                   rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = warp_validate(x, flow, N, C, H, W, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "warp_bwd: dy is required");
    if (dx && o.algo == RS_ALGO_GATHER)
        return fail(RS_ERR_FLAG, "warp_bwd: GATHER invalid (arbitrary flow has no bounded inverse)");
    if (dx && o.deterministic && (o.algo == RS_ALGO_SCATTER_ATOMIC || o.algo == RS_ALGO_SCATTER_PRIV))
        return fail(RS_ERR_FLAG, "warp_bwd: SCATTER_ATOMIC / SCATTER_PRIV are atomic paths (not deterministic)");
    if (!dx && !dflow) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{x, sizeof(float) * (size_t)C * H * W, true, false},
                              {flow, sizeof(float) * 2 * (size_t)H * W, true, false},
                              {dy, sizeof(float) * (size_t)C * H * W, true, false},
                              {dx, sizeof(float) * (size_t)C * H * W, false, true},
                              {dflow, sizeof(float) * 2 * (size_t)H * W, false, true}};
    const bool det = o.deterministic && dx;
    return run_batched(N, args, s, workspace, ws_bytes, [&](int n) { return rs::warp_ws_bytes(n, C, H, W, det); },
                       [&](int, int nc, void **p, cudaStream_t t, void *ws) {
                           rs::WarpArgs a{};
                           a.x = (const float *)p[0];
                           a.flow = (const float *)p[1];
                           a.dy = (const float *)p[2];
                           a.dx = (float *)p[3];
                           a.dflow = (float *)p[4];
                           a.N = nc; a.C = C; a.H = H; a.W = W;
                           a.border = o.padding == RS_PAD_BORDER;
                           return rs::warp_bwd_launch(a, o.algo, o.deterministic, ws,
                                                      rs::warp_ws_bytes(nc, C, H, W, det), t);
                       });
}

// ------------------------------------------------------------------------------ bslice
static rs_status bslice_validate(const float *grid, const float *guide, const float *x, int N, int H,
                                 int W, int D, int Gh, int Gw, const rs_opts &o) {
    if (!grid || !guide || !x) return fail(RS_ERR_NULL, "bslice: grid, guide and x are required");
    if (!pos(N) || !pos(H) || !pos(W) || !pos(D) || !pos(Gh) || !pos(Gw))
        return fail(RS_ERR_SHAPE, "bslice: dims must be positive (N=%d H=%d W=%d D=%d Gh=%d Gw=%d)",
                    N, H, W, D, Gh, Gw);
    if (H > 65535 || W > 65535) return fail(RS_ERR_SHAPE, "bslice: H, W must be <= 65535");
    if ((long long)N * (Gh + 1) * (Gw + 1) * 4 >= (1LL << 31))
        return fail(RS_ERR_SHAPE, "bslice: too many dual-cell tiles per launch (split the batch)");
    return check_opts(o);
}

rs_status bslice_fwd(const float *grid, const float *guide, const float *x, int N, int H, int W,
                     int D, int Gh, int Gw, const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = bslice_validate(grid, guide, x, N, H, W, D, Gh, Gw, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "bslice_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{grid, sizeof(float) * 12 * (size_t)D * Gh * Gw, true, false},
                              {guide, sizeof(float) * (size_t)H * W, true, false},
                              {x, sizeof(float) * 3 * (size_t)H * W, true, false},
                              {y, sizeof(float) * 3 * (size_t)H * W, false, true}};
    return run_batched(N, args, s, nullptr, 0, [](int) { return (size_t)0; },
                       [&](int, int nc, void **p, cudaStream_t t, void *) {
                           rs::BsliceArgs a{};
                           a.grid = (const float *)p[0];
                           a.guide = (const float *)p[1];
                           a.x = (const float *)p[2];
                           a.y = (float *)p[3];
                           a.N = nc; a.H = H; a.W = W; a.D = D; a.Gh = Gh; a.Gw = Gw;
                           return rs::bslice_fwd_launch(a, t);
                       });
}

rs_status bslice_bwd(const float *grid, const float *guide, const float *x, const float *dy, int N,
                     int H, int W, int D, int Gh, int Gw, const rs_opts *opts, float *dgrid,
                     float *dguide, float *dx, void *workspace, size_t ws_bytes,
                     rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = bslice_validate(grid, guide, x, N, H, W, D, Gh, Gw, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "bslice_bwd: dy is required");
    if (dgrid && o.algo == RS_ALGO_SCATTER_ATOMIC && o.deterministic)
        return fail(RS_ERR_FLAG, "bslice_bwd: SCATTER_ATOMIC is not deterministic");
    if (!dgrid && !dguide && !dx) return ok();
    const bool det = o.deterministic && dgrid;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<TArg> args = {{grid, sizeof(float) * 12 * (size_t)D * Gh * Gw, true, false},
                              {guide, sizeof(float) * (size_t)H * W, true, false},
                              {x, sizeof(float) * 3 * (size_t)H * W, true, false},
                              {dy, sizeof(float) * 3 * (size_t)H * W, true, false},
                              {dgrid, sizeof(float) * 12 * (size_t)D * Gh * Gw, false, true},
                              {dguide, sizeof(float) * (size_t)H * W, false, true},
                              {dx, sizeof(float) * 3 * (size_t)H * W, false, true}};
    return run_batched(N, args, s, workspace, ws_bytes,
                       [&](int n) { return rs::bslice_bwd_ws_bytes(n, H, W, D, Gh, Gw, det); },
                       [&](int, int nc, void **p, cudaStream_t t, void *ws) {
                           rs::BsliceArgs a{};
                           a.grid = (const float *)p[0];
                           a.guide = (const float *)p[1];
                           a.x = (const float *)p[2];
                           a.dy = (const float *)p[3];
                           a.dgrid = (float *)p[4];
                           a.dguide = (float *)p[5];
                           a.dx = (float *)p[6];
                           a.N = nc; a.H = H; a.W = W; a.D = D; a.Gh = Gh; a.Gw = Gw;
                           return rs::bslice_bwd_launch(a, o.algo, o.deterministic, ws,
                                                        rs::bslice_bwd_ws_bytes(nc, H, W, D, Gh, Gw, det), t);
                       });
}


// ------------------------------------------------------------------------------ conv
static rs_status conv_validate(const float *x, const float *k, int N, int Ci, int Co, int H, int W,
                               int kh, int kw, const rs_opts &o) {
    if (!x || !k) return fail(RS_ERR_NULL, "conv: x and k are required");
    if (!pos(N) || !pos(Ci) || !pos(Co) || !pos(H) || !pos(W) || !pos(kh) || !pos(kw))
        return fail(RS_ERR_SHAPE, "conv: dims must be positive (N=%d Ci=%d Co=%d H=%d W=%d kh=%d kw=%d)", N,
                    Ci, Co, H, W, kh, kw);
    if (N > 65535 || (long long)H * W >= (1LL << 31) || (long long)Co * H * W >= (1LL << 40))
        return fail(RS_ERR_SHAPE, "conv: N <= 65535 and H*W < 2^31");
    if (!rs::conv_shape_ok(Ci, Co, kh, kw))
        return fail(RS_ERR_SHAPE, "conv: kh, kw must be <= 7 and Ci input windows must fit in shared memory");
    if (!is_device_ptr(x) || !is_device_ptr(k))
        return fail(RS_ERR_FLAG, "conv: device pointers only");
    return check_opts(o);
}

rs_status conv_fwd(const float *x, const float *k, int N, int Ci, int Co, int H, int W, int kh, int kw,
                   const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = conv_validate(x, k, N, Ci, Co, H, W, kh, kw, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "conv_fwd: y is required");
    if (!is_device_ptr(y)) return fail(RS_ERR_FLAG, "conv: device pointers only");
    rs::ConvArgs a{};
    a.x = x; a.k = k; a.y = y;
    a.N = N; a.Ci = Ci; a.Co = Co; a.H = H; a.W = W; a.kh = kh; a.kw = kw;
    return launched(rs::conv_fwd_launch(a, (cudaStream_t)stream), "conv_fwd");
}

rs_status conv_bwd(const float *x, const float *k, const float *dy, int N, int Ci, int Co, int H, int W,
                   int kh, int kw, const rs_opts *opts, float *dx, float *dk, void *workspace, size_t ws_bytes,
                   rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = conv_validate(x, k, N, Ci, Co, H, W, kh, kw, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "conv_bwd: dy is required");
    if (dx && o.algo == RS_ALGO_SCATTER_PRIV)
        return fail(RS_ERR_FLAG, "conv_bwd: SCATTER_PRIV is not implemented for the conv layer");
    if (dx && o.algo == RS_ALGO_SCATTER_ATOMIC && o.deterministic)
        return fail(RS_ERR_FLAG, "conv_bwd: the atomic scatter is not deterministic");
    if (!is_device_ptr(dy) || (dx && !is_device_ptr(dx)) || (dk && !is_device_ptr(dk)))
        return fail(RS_ERR_FLAG, "conv: device pointers only");
    if (!dx && !dk) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    rs::ConvArgs a{};
    a.x = x; a.k = k; a.dy = dy; a.dx = dx; a.dk = dk;
    a.N = N; a.Ci = Ci; a.Co = Co; a.H = H; a.W = W; a.kh = kh; a.kw = kw;
    const size_t need = dk ? rs::conv_ws_bytes(N, Ci, Co, H, W, kh, kw) : 0;
    void *ws = workspace;
    bool own = false;
    if (need && (!ws || ws_bytes < need)) {
        cudaError_t e = lib_malloc(&ws, need, s);
        if (e != cudaSuccess) return fail(RS_ERR_WORKSPACE, "workspace cudaMallocAsync(%zu): %s", need, cudaGetErrorString(e));
        own = true;
        ws_bytes = need;
    }
    cudaError_t e = rs::conv_bwd_launch(a, o.algo, ws, ws_bytes, s);
    if (own) cudaFreeAsync(ws, s);
    return launched(e, "conv_bwd");
}

// ------------------------------------------------------------------------------ f4
rs_status convloss_grad(const float *in, const float *k, const float *target, int N, int H, int W, int kh,
                        int kw, rs_schedule schedule, float *d_in, void *workspace, size_t ws_bytes,
                        rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    if (!in || !k || !target || !d_in) return fail(RS_ERR_NULL, "convloss_grad: in, k, target, d_in are required");
    if (!pos(N) || !pos(H) || !pos(W) || !pos(kh) || !pos(kw) || kh > 7 || kw > 7)
        return fail(RS_ERR_SHAPE, "convloss_grad: positive dims, 1 <= kh, kw <= 7 (N=%d H=%d W=%d kh=%d kw=%d)", N,
                    H, W, kh, kw);
    if (N > 65535 || (long long)H * W >= (1LL << 31)) return fail(RS_ERR_SHAPE, "convloss_grad: H*W < 2^31");
    if (schedule != RS_SCHED_ROOT && schedule != RS_SCHED_INLINE && schedule != RS_SCHED_AT)
        return fail(RS_ERR_FLAG, "convloss_grad: unknown schedule %d", (int)schedule);
    if (!is_device_ptr(in) || !is_device_ptr(target) || !is_device_ptr(d_in))
        return fail(RS_ERR_FLAG, "convloss_grad: in, target, d_in must be device pointers");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t need = schedule == RS_SCHED_ROOT ? rs::convloss_ws_bytes(N, H, W) : 0;
    void *ws = workspace;
    bool own = false;
    if (need && (!ws || ws_bytes < need)) {
        cudaError_t e = lib_malloc(&ws, need, s);
        if (e != cudaSuccess) return fail(RS_ERR_WORKSPACE, "workspace cudaMallocAsync(%zu): %s", need, cudaGetErrorString(e));
        own = true;
    }
    cudaError_t e = rs::convloss_grad_launch(in, k, target, N, H, W, kh, kw, (int)schedule, d_in, ws, s);
    if (own) cudaFreeAsync(ws, s);
    return launched(e, "convloss_grad");
}

static rs_status up4_check(const void *a, const void *b, int N, int C, int H, int W) {
    if (!a || !b) return fail(RS_ERR_NULL, "upsample4: both tensors are required");
    if (!pos(N) || !pos(C) || !pos(H) || !pos(W) || 16LL * N * C * H * W >= (1LL << 40))
        return fail(RS_ERR_SHAPE, "upsample4: positive dims");
    if (!is_device_ptr(a) || !is_device_ptr(b)) return fail(RS_ERR_FLAG, "upsample4: device pointers only");
    return RS_OK;
}

rs_status upsample4_fwd(const float *x, int N, int C, int H, int W, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    rs_status st = up4_check(x, y, N, C, H, W);
    if (st != RS_OK) return st;
    return launched(rs::upsample4_launch(x, y, N, C, H, W, false, (cudaStream_t)stream), "upsample4_fwd");
}

rs_status upsample4_bwd(const float *dy, int N, int C, int H, int W, float *dx, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    rs_status st = up4_check(dy, dx, N, C, H, W);
    if (st != RS_OK) return st;
    return launched(rs::upsample4_launch(dy, dx, N, C, H, W, true, (cudaStream_t)stream), "upsample4_bwd");
}

// ------------------------------------------------------------------------------ f3
static rs_status var_check(const rs_opts &o, bool bwd, bool has_dx, std::initializer_list<const void *> ptrs,
                           bool has_gather = false) {
    rs_status st = check_opts(o);
    if (st != RS_OK) return st;
    if (o.padding != RS_PAD_ZEROS) return fail(RS_ERR_FLAG, "stn variants: zeros padding only");
    if (bwd && has_dx && o.algo == RS_ALGO_SCATTER_PRIV)
        return fail(RS_ERR_FLAG, "stn variants: SCATTER_PRIV is not implemented");
    if (bwd && has_dx && !has_gather && o.algo == RS_ALGO_GATHER)
        return fail(RS_ERR_FLAG, "stn3d / lanczos: no gather form of d_input (scatter only)");
    if (bwd && has_dx && o.algo == RS_ALGO_SCATTER_ATOMIC && o.deterministic)
        return fail(RS_ERR_FLAG, "stn variants: the atomic scatter is not deterministic");
    for (const void *p : ptrs)
        if (p && !is_device_ptr(p)) return fail(RS_ERR_FLAG, "stn variants: device pointers only");
    return RS_OK;
}

extern "C++" {
template <class F>
rs_status with_ws(size_t need, void *workspace, size_t ws_bytes, cudaStream_t s, F &&f, const char *what) {
    void *ws = workspace;
    bool own = false;
    if (need && (!ws || ws_bytes < need)) {
        cudaError_t e = lib_malloc(&ws, need, s);
        if (e != cudaSuccess) return fail(RS_ERR_WORKSPACE, "workspace cudaMallocAsync(%zu): %s", need, cudaGetErrorString(e));
        own = true;
    }
    cudaError_t e = f(ws);
    if (own) cudaFreeAsync(ws, s);
    return launched(e, what);
}
}  // extern "C++"

rs_status stn_bicubic_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho, int Wo,
                          const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "stn_bicubic_fwd: y is required");
    if ((st = var_check(o, false, false, {x, theta, y})) != RS_OK) return st;
    rs::StnArgs a{};
    a.x = x; a.theta = theta; a.y = y;
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo; a.ac = o.align_corners;
    return launched(rs::stn_bicubic_launch(a, false, 0, false, nullptr, (cudaStream_t)stream), "stn_bicubic_fwd");
}

rs_status stn_bicubic_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H, int W, int Ho,
                          int Wo, const rs_opts *opts, float *dx, float *dtheta, void *workspace, size_t ws_bytes,
                          rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "stn_bicubic_bwd: dy is required");
    if ((st = var_check(o, true, dx != nullptr, {x, theta, dy, dx, dtheta}, true)) != RS_OK) return st;
    if (!dx && !dtheta) return ok();
    rs::StnArgs a{};
    a.x = x; a.theta = theta; a.dy = dy; a.dx = dx; a.dtheta = dtheta;
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo; a.ac = o.align_corners;
    cudaStream_t s = (cudaStream_t)stream;
    const bool det = o.deterministic && dx;
    return with_ws(rs::stn_bicubic_ws_bytes(N, C, H, W, Ho, Wo, det), workspace, ws_bytes, s,
                   [&](void *ws) {
                       return rs::stn_bicubic_launch(a, true, (int)o.algo, det, ws, s);
                   },
                   "stn_bicubic_bwd");
}

static rs_status stn3d_validate(const float *x, const float *theta, int N, int C, int D, int H, int W, int Do, int Ho,
                                int Wo, const rs_opts &o) {
    if (!x || !theta) return fail(RS_ERR_NULL, "stn3d: x and theta are required");
    if (!pos(N) || !pos(C) || !pos(D) || !pos(H) || !pos(W) || !pos(Do) || !pos(Ho) || !pos(Wo))
        return fail(RS_ERR_SHAPE, "stn3d: dims must be positive");
    if (o.align_corners && (Do < 2 || Ho < 2 || Wo < 2))
        return fail(RS_ERR_SHAPE, "stn3d: align_corners=1 needs Do, Ho, Wo >= 2");
    if (N > 65535 || (long long)Do * Ho * Wo >= (1LL << 31) || (long long)D * H * W >= (1LL << 40))
        return fail(RS_ERR_SHAPE, "stn3d: N <= 65535 and Do*Ho*Wo < 2^31");
    return RS_OK;
}

rs_status stn3d_fwd(const float *x, const float *theta, int N, int C, int D, int H, int W, int Do, int Ho, int Wo,
                    const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn3d_validate(x, theta, N, C, D, H, W, Do, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "stn3d_fwd: y is required");
    if ((st = var_check(o, false, false, {x, theta, y})) != RS_OK) return st;
    return launched(rs::stn3d_launch(x, theta, nullptr, y, nullptr, nullptr, N, C, D, H, W, Do, Ho, Wo,
                                     o.align_corners, false, false, nullptr, (cudaStream_t)stream),
                    "stn3d_fwd");
}

rs_status stn3d_bwd(const float *x, const float *theta, const float *dy, int N, int C, int D, int H, int W, int Do,
                    int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta, void *workspace, size_t ws_bytes,
                    rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn3d_validate(x, theta, N, C, D, H, W, Do, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "stn3d_bwd: dy is required");
    if ((st = var_check(o, true, dx != nullptr, {x, theta, dy, dx, dtheta})) != RS_OK) return st;
    if (!dx && !dtheta) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    const bool det = o.deterministic && dx;
    return with_ws(rs::stn3d_ws_bytes(N, C, D, H, W, Do, Ho, Wo, det), workspace, ws_bytes, s,
                   [&](void *ws) {
                       return rs::stn3d_launch(x, theta, dy, nullptr, dx, dtheta, N, C, D, H, W, Do, Ho, Wo,
                                               o.align_corners, true, det, ws, s);
                   },
                   "stn3d_bwd");
}

rs_status stn_lanczos_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho, int Wo,
                          const rs_opts *opts, float *y, rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "stn_lanczos_fwd: y is required");
    if ((st = var_check(o, false, false, {x, theta, y})) != RS_OK) return st;
    rs::StnArgs a{};
    a.x = x; a.theta = theta; a.y = y;
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo; a.ac = o.align_corners;
    return launched(rs::stn_lanczos_launch(a, false, false, nullptr, (cudaStream_t)stream), "stn_lanczos_fwd");
}

rs_status stn_lanczos_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H, int W, int Ho,
                          int Wo, const rs_opts *opts, float *dx, float *dtheta, void *workspace, size_t ws_bytes,
                          rs_stream_t stream) {
    DeviceGuard dg_((cudaStream_t)stream);
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "stn_lanczos_bwd: dy is required");
    if ((st = var_check(o, true, dx != nullptr, {x, theta, dy, dx, dtheta})) != RS_OK) return st;
    if (!dx && !dtheta) return ok();
    rs::StnArgs a{};
    a.x = x; a.theta = theta; a.dy = dy; a.dx = dx; a.dtheta = dtheta;
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo; a.ac = o.align_corners;
    cudaStream_t s = (cudaStream_t)stream;
    const bool det = o.deterministic && dx;
    return with_ws(rs::stn_lanczos_ws_bytes(N, C, H, W, Ho, Wo, det), workspace, ws_bytes, s,
                   [&](void *ws) { return rs::stn_lanczos_launch(a, true, det, ws, s); }, "stn_lanczos_bwd");
}

}  // extern "C"
