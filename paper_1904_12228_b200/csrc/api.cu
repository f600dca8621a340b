// api.cu — the extern "C" boundary declared in include/rsgrad.h.
//
// Responsibilities: argument validation, option defaults, host-pointer staging
// (stream-ordered temporaries), workspace provisioning, error reporting through
// a thread-local string, and dispatch to the per-layer launchers.  No compute.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

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

// Host-or-device pointer staging.  Every buffer the call touches is registered;
// host ones get a stream-ordered device temporary.
class Stager {
   public:
    explicit Stager(cudaStream_t s) : s_(s) {}
    ~Stager() {
        for (auto &e : ents_)
            if (e.dev && e.owned) cudaFreeAsync(e.dev, s_);
    }
    // returns the device-visible pointer (nullptr stays nullptr)
    template <typename T>
    T *in(const T *p, size_t count, rs_status &st) {
        return (T *)stage((void *)p, count * sizeof(T), true, false, st);
    }
    template <typename T>
    T *out(T *p, size_t count, rs_status &st) {
        return (T *)stage((void *)p, count * sizeof(T), false, true, st);
    }
    void *scratch(size_t bytes, rs_status &st) {
        void *d = nullptr;
        cudaError_t e = cudaMallocAsync(&d, bytes ? bytes : 1, s_);
        if (e != cudaSuccess) {
            st = fail(RS_ERR_WORKSPACE, "workspace cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
            return nullptr;
        }
        ents_.push_back({nullptr, d, 0, false, true});
        return d;
    }
    // copy staged outputs back to the caller's host buffers
    rs_status finish() {
        for (auto &e : ents_) {
            if (e.host && e.is_out) {
                cudaError_t c = cudaMemcpyAsync(e.host, e.dev, e.bytes, cudaMemcpyDeviceToHost, s_);
                if (c != cudaSuccess)
                    return fail(RS_ERR_CUDA, "D2H copy: %s", cudaGetErrorString(c));
            }
        }
        return RS_OK;
    }
    size_t h2d_bytes() const { return h2d_; }

   private:
    struct Ent {
        void *host;
        void *dev;
        size_t bytes;
        bool is_out;
        bool owned;
    };
    void *stage(void *p, size_t bytes, bool is_in, bool is_out, rs_status &st) {
        if (!p) return nullptr;
        cudaPointerAttributes at;
        cudaError_t e = cudaPointerGetAttributes(&at, p);
        if (e != cudaSuccess) {
            cudaGetLastError();  // clear
            at.type = cudaMemoryTypeUnregistered;
        }
        if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return p;
        void *d = nullptr;
        e = cudaMallocAsync(&d, bytes ? bytes : 1, s_);
        if (e != cudaSuccess) {
            st = fail(RS_ERR_CUDA, "staging cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
            return nullptr;
        }
        ents_.push_back({p, d, bytes, is_out, true});
        if (is_in) {
            e = cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s_);
            if (e != cudaSuccess) {
                st = fail(RS_ERR_CUDA, "H2D copy: %s", cudaGetErrorString(e));
                return nullptr;
            }
            h2d_ += bytes;
        }
        return d;
    }
    cudaStream_t s_;
    std::vector<Ent> ents_;
    size_t h2d_ = 0;
};

rs_status launched(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return ok();
}

bool pos(int v) { return v > 0; }

}  // namespace

extern "C" {

const char *rsgrad_last_error(void) { return rs::g_err; }

const char *rsgrad_version(void) { return "rsgrad 0.1.0 sm_100a"; }

unsigned long long rsgrad_launch_count(int reset) {
    unsigned long long v = rs::g_launches;
    if (reset) rs::g_launches = 0;
    return v;
}

size_t rsgrad_bwd_workspace_bytes(int layer, int N, int C, int H, int W, int Ho, int Wo, int D,
                                  int Gh, int Gw, const rs_opts *opts) {
    (void)opts;
    switch (layer) {
        case 0:
            if (!pos(N) || !pos(Ho) || !pos(Wo)) return 0;
            return rs::stn_ws_bytes(N, C, H, W, Ho, Wo);
        case 1:
            return rs::warp_ws_bytes(N, C, H, W);
        case 2:
            if (!pos(N) || !pos(H) || !pos(W) || !pos(D) || !pos(Gh) || !pos(Gw)) return 0;
            return rs::bslice_ws_bytes(N, H, W, D, Gh, Gw);
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
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "stn_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::StnArgs a{};
    a.x = sg.in(x, (size_t)N * C * H * W, st);
    a.theta = sg.in(theta, (size_t)N * 6, st);
    a.y = sg.out(y, (size_t)N * C * Ho * Wo, st);
    if (st != RS_OK) return st;
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
    a.ac = o.align_corners;
    a.border = o.padding == RS_PAD_BORDER;
    st = launched(rs::stn_fwd_launch(a, s), "stn_fwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
}

rs_status stn_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H, int W,
                  int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta, void *workspace,
                  size_t ws_bytes, rs_stream_t stream) {
    const rs_opts o = resolve(opts);
    rs_status st = stn_validate(x, theta, N, C, H, W, Ho, Wo, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "stn_bwd: dy is required");
    const bool border = o.padding == RS_PAD_BORDER;
    if (dx && border && o.algo == RS_ALGO_GATHER)
        return fail(RS_ERR_FLAG, "stn_bwd: GATHER needs zeros padding (border clamp has no bounded inverse)");
    if (dx && border && o.deterministic)
        return fail(RS_ERR_FLAG, "stn_bwd: no deterministic d_input path with border padding");
    if (dx && o.algo == RS_ALGO_SCATTER_PRIV)
        return fail(RS_ERR_FLAG, "stn_bwd: SCATTER_PRIV not implemented for STN (use AUTO/GATHER/SCATTER_ATOMIC)");
    if (dx && o.algo == RS_ALGO_SCATTER_ATOMIC && o.deterministic)
        return fail(RS_ERR_FLAG, "stn_bwd: SCATTER_ATOMIC is not deterministic");
    if (!dx && !dtheta) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::StnArgs a{};
    a.x = sg.in(x, (size_t)N * C * H * W, st);
    a.theta = sg.in(theta, (size_t)N * 6, st);
    a.dy = sg.in(dy, (size_t)N * C * Ho * Wo, st);
    a.dx = sg.out(dx, (size_t)N * C * H * W, st);
    a.dtheta = sg.out(dtheta, (size_t)N * 6, st);
    if (st != RS_OK) return st;
    const size_t need = rs::stn_ws_bytes(N, C, H, W, Ho, Wo);
    void *ws = workspace;
    if (!ws || ws_bytes < need) {
        ws = sg.scratch(need, st);
        if (st != RS_OK) return st;
    }
    a.N = N; a.C = C; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
    a.ac = o.align_corners;
    a.border = border;
    st = launched(rs::stn_bwd_launch(a, o.algo, o.deterministic, ws, need, s), "stn_bwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
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
    const rs_opts o = resolve(opts);
    rs_status st = warp_validate(x, flow, N, C, H, W, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "warp_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::WarpArgs a{};
    a.x = sg.in(x, (size_t)N * C * H * W, st);
    a.flow = sg.in(flow, (size_t)N * 2 * H * W, st);
    a.y = sg.out(y, (size_t)N * C * H * W, st);
    if (st != RS_OK) return st;
    a.N = N; a.C = C; a.H = H; a.W = W;
    a.border = o.padding == RS_PAD_BORDER;
    st = launched(rs::warp_fwd_launch(a, s), "warp_fwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
}

rs_status warp_bwd(const float *x, const float *flow, const float *dy, int N, int C, int H, int W,
                   const rs_opts *opts, float *dx, float *dflow, void *workspace, size_t ws_bytes,
                   rs_stream_t stream) {
    const rs_opts o = resolve(opts);
    rs_status st = warp_validate(x, flow, N, C, H, W, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "warp_bwd: dy is required");
    if (dx && o.algo == RS_ALGO_GATHER)
        return fail(RS_ERR_FLAG, "warp_bwd: GATHER invalid (arbitrary flow has no bounded inverse)");
    if (dx && o.algo == RS_ALGO_SCATTER_PRIV)
        return fail(RS_ERR_FLAG, "warp_bwd: SCATTER_PRIV not implemented yet (use AUTO/SCATTER_ATOMIC)");
    if (dx && o.deterministic)
        return fail(RS_ERR_FLAG, "warp_bwd: no deterministic d_input path (atomic scatter)");
    if (!dx && !dflow) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::WarpArgs a{};
    a.x = sg.in(x, (size_t)N * C * H * W, st);
    a.flow = sg.in(flow, (size_t)N * 2 * H * W, st);
    a.dy = sg.in(dy, (size_t)N * C * H * W, st);
    a.dx = sg.out(dx, (size_t)N * C * H * W, st);
    a.dflow = sg.out(dflow, (size_t)N * 2 * H * W, st);
    if (st != RS_OK) return st;
    a.N = N; a.C = C; a.H = H; a.W = W;
    a.border = o.padding == RS_PAD_BORDER;
    st = launched(rs::warp_bwd_launch(a, o.algo, o.deterministic, workspace, ws_bytes, s),
                  "warp_bwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
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
    const rs_opts o = resolve(opts);
    rs_status st = bslice_validate(grid, guide, x, N, H, W, D, Gh, Gw, o);
    if (st != RS_OK) return st;
    if (!y) return fail(RS_ERR_NULL, "bslice_fwd: y is required");
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::BsliceArgs a{};
    a.grid = sg.in(grid, (size_t)N * 12 * D * Gh * Gw, st);
    a.guide = sg.in(guide, (size_t)N * H * W, st);
    a.x = sg.in(x, (size_t)N * 3 * H * W, st);
    a.y = sg.out(y, (size_t)N * 3 * H * W, st);
    if (st != RS_OK) return st;
    a.N = N; a.H = H; a.W = W; a.D = D; a.Gh = Gh; a.Gw = Gw;
    st = launched(rs::bslice_fwd_launch(a, s), "bslice_fwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
}

rs_status bslice_bwd(const float *grid, const float *guide, const float *x, const float *dy, int N,
                     int H, int W, int D, int Gh, int Gw, const rs_opts *opts, float *dgrid,
                     float *dguide, float *dx, void *workspace, size_t ws_bytes,
                     rs_stream_t stream) {
    const rs_opts o = resolve(opts);
    rs_status st = bslice_validate(grid, guide, x, N, H, W, D, Gh, Gw, o);
    if (st != RS_OK) return st;
    if (!dy) return fail(RS_ERR_NULL, "bslice_bwd: dy is required");
    if (dgrid && o.algo == RS_ALGO_SCATTER_ATOMIC && o.deterministic)
        return fail(RS_ERR_FLAG, "bslice_bwd: SCATTER_ATOMIC is not deterministic");
    if (dgrid && o.deterministic && rs::bslice_ws_bytes(N, H, W, D, Gh, Gw) == 0)
        return fail(RS_ERR_FLAG, "bslice_bwd: shape needs the atomic d_grid path (cells < 8 px); not deterministic");
    if (!dgrid && !dguide && !dx) return ok();
    cudaStream_t s = (cudaStream_t)stream;
    Stager sg(s);
    rs::BsliceArgs a{};
    a.grid = sg.in(grid, (size_t)N * 12 * D * Gh * Gw, st);
    a.guide = sg.in(guide, (size_t)N * H * W, st);
    a.x = sg.in(x, (size_t)N * 3 * H * W, st);
    a.dy = sg.in(dy, (size_t)N * 3 * H * W, st);
    a.dgrid = sg.out(dgrid, (size_t)N * 12 * D * Gh * Gw, st);
    a.dguide = sg.out(dguide, (size_t)N * H * W, st);
    a.dx = sg.out(dx, (size_t)N * 3 * H * W, st);
    if (st != RS_OK) return st;
    a.N = N; a.H = H; a.W = W; a.D = D; a.Gh = Gh; a.Gw = Gw;
    size_t need = rs::bslice_ws_bytes(N, H, W, D, Gh, Gw);
    void *ws = workspace;
    if (need && (!ws || ws_bytes < need)) {
        ws = sg.scratch(need, st);
        if (st != RS_OK) return st;
    }
    st = launched(rs::bslice_bwd_launch(a, o.algo, o.deterministic, ws, need, s), "bslice_bwd launch");
    if (st != RS_OK) return st;
    return sg.finish() == RS_OK ? ok() : RS_ERR_CUDA;
}

}  // extern "C"
