// warp.cu — FlowNet 2.0 per-pixel warp, forward and adjoint, sm_100a.
//
// Kernels
//   warp_fwd_kernel   one thread per pixel: coordinate x + u(x) in fp64, bilinear
//                     gather over all channels.
//   warp_bwd_kernel   one thread per pixel: d_flow is a pure gather (G and the X
//                     taps); d_input is the reversed gather, which for an
//                     arbitrary flow field has no bounded inverse, so it is
//                     "a general scatter using atomics": fp32
//                     red.global.add into a zero-filled dx (AUTO, SCATTER_ATOMIC).
//   warp_bwd_win      variant (RSGRAD_WARP_BWD=winR,NW,IT): per-warp shared windows
//                     flushed by red.v4 (measured slower).
//   SCATTER_PRIV goes through the staged-footprint output tile of stn.cu (flow mode).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace rs {
namespace {

#ifndef RS_WARP_T
#define RS_WARP_T 128
#endif
constexpr int kThreads = RS_WARP_T;  // per-pixel kernels: 128 measured vs 256: fwd 0.771 vs 0.809 ms (64 samples)

#ifndef RS_TAP_HINT
#define RS_TAP_HINT 1
#endif
#if RS_TAP_HINT
#define TAPLD(p) ldg_tap(p)
#else
#define TAPLD(p) __ldg(p)
#endif

struct Tap {
    long long o00;
    int x0, y0;  // floor cell
    float w00, w01, w10, w11;
    float fx, fy;
    bool k00, k01, k10, k11;
};

RS_DEV Tap warp_tap(const WarpArgs &a, int x, int y, float u, float v, float &cgx, float &cgy) {
    double ix = __dadd_rn((double)x, (double)u);
    double iy = __dadd_rn((double)y, (double)v);
    cgx = 1.f;
    cgy = 1.f;
    if (a.border) {
        ix = clamp_coord(ix, a.W, cgx);
        iy = clamp_coord(iy, a.H, cgy);
    }
    const Cell cx = cell_of(ix), cy = cell_of(iy);
    const bool x0ok = cx.i0 >= 0 && cx.i0 < a.W, x1ok = cx.i0 + 1 >= 0 && cx.i0 + 1 < a.W;
    const bool y0ok = cy.i0 >= 0 && cy.i0 < a.H, y1ok = cy.i0 + 1 >= 0 && cy.i0 + 1 < a.H;
    Tap t;
    t.fx = cx.f;
    t.fy = cy.f;
    const float wx0 = 1.f - cx.f, wy0 = 1.f - cy.f;
    t.w00 = wy0 * wx0;
    t.w01 = wy0 * cx.f;
    t.w10 = cy.f * wx0;
    t.w11 = cy.f * cx.f;
    t.k00 = y0ok && x0ok;
    t.k01 = y0ok && x1ok;
    t.k10 = y1ok && x0ok;
    t.k11 = y1ok && x1ok;
    t.o00 = (long long)cy.i0 * a.W + cx.i0;
    t.x0 = cx.i0;
    t.y0 = cy.i0;
    return t;
}

// grid = (ceil(H*W / 256), N): sample from blockIdx.y, 32-bit offsets inside a sample
// (H*W < 2^31 is validated by the API), row from a reciprocal-multiply division.
__global__ void __launch_bounds__(kThreads) warp_fwd_kernel(WarpArgs a, double invW) {
    const int HW = a.H * a.W;
    const int rem = blockIdx.x * kThreads + threadIdx.x;
    if (rem >= HW) return;
    const int n = blockIdx.y;
    const int y = fast_div(rem, a.W, invW), x = rem - y * a.W;
    const float *fp = a.flow + (long long)n * 2 * HW + rem;
    const float u = ldg_stream(fp), v = ldg_stream(fp + HW);
    float cgx, cgy;
    const Tap t = warp_tap(a, x, y, u, v, cgx, cgy);
    const float *xp = a.x + (long long)n * a.C * HW;
    float *yp = a.y + (long long)n * a.C * HW + rem;
    const int o00 = (int)t.o00;
#pragma unroll 3
    for (int c = 0; c < a.C; c++) {
        const float *p = xp + o00;
        float r = 0.f;
        if (t.k00) r = fmaf(t.w00, TAPLD(p), r);
        if (t.k01) r = fmaf(t.w01, TAPLD(p + 1), r);
        if (t.k10) r = fmaf(t.w10, TAPLD(p + a.W), r);
        if (t.k11) r = fmaf(t.w11, TAPLD(p + a.W + 1), r);
        *yp = r;
        xp += HW;
        yp += HW;
    }
}

__global__ void __launch_bounds__(kThreads) warp_bwd_kernel(WarpArgs a, double invW) {
    const int HW = a.H * a.W;
    const int rem0 = blockIdx.x * kThreads + threadIdx.x;
    const bool live = rem0 < HW;
    const int rem = live ? rem0 : HW - 1;  // tail lanes shadow the last pixel (all work masked)
    const int n = blockIdx.y;
    const int y = fast_div(rem, a.W, invW), x = rem - y * a.W;
    const float *fp = a.flow + (long long)n * 2 * HW + rem;
    const float u = ldg_stream(fp), v = ldg_stream(fp + HW);
    float cgx, cgy;
    Tap t = warp_tap(a, x, y, u, v, cgx, cgy);
    if (!live) t.k00 = t.k01 = t.k10 = t.k11 = false;
    const int o00 = (int)t.o00;
    const float *xp = a.x + (long long)n * a.C * HW + o00;
    float *dxp = a.dx ? a.dx + (long long)n * a.C * HW + o00 : nullptr;
    // lane l absorbs lane l-1's right taps if they are the same addresses (o00 one apart,
    // same sample: blocks never straddle samples, and a row step changes o00 by W)
    const int lane = threadIdx.x & 31;
    const int o_prev = __shfl_up_sync(0xffffffffu, o00, 1);
    const bool k01_prev = __shfl_up_sync(0xffffffffu, (int)t.k01, 1) != 0;
    const bool k11_prev = __shfl_up_sync(0xffffffffu, (int)t.k11, 1) != 0;
    const bool absorb = lane > 0 && o_prev + 1 == o00 && k01_prev == t.k00 && k11_prev == t.k10;
    const bool given = __shfl_down_sync(0xffffffffu, (int)absorb, 1) != 0 && lane < 31;
    const float *gp = a.dy + (long long)n * a.C * HW + rem;
    float dix = 0.f, diy = 0.f;
    for (int c = 0; c < a.C; c++) {
        const float g = ldg_stream(gp);
        if (a.dflow) {
            const float v00 = t.k00 ? TAPLD(xp) : 0.f, v01 = t.k01 ? TAPLD(xp + 1) : 0.f;
            const float v10 = t.k10 ? TAPLD(xp + a.W) : 0.f, v11 = t.k11 ? TAPLD(xp + a.W + 1) : 0.f;
            dix = fmaf(g, fmaf(1.f - t.fy, v01 - v00, t.fy * (v11 - v10)), dix);
            diy = fmaf(g, fmaf(1.f - t.fx, v10 - v00, t.fx * (v11 - v01)), diy);
        }
        if (dxp) {
            // merge with the left neighbour lane when its right taps are our left taps
            // (same row, floor cell one to the left): about half the reds for smooth flow
            const float r01 = __shfl_up_sync(0xffffffffu, t.w01 * g, 1);
            const float r11 = __shfl_up_sync(0xffffffffu, t.w11 * g, 1);
            const float l00 = t.w00 * g + (absorb ? r01 : 0.f), l10 = t.w10 * g + (absorb ? r11 : 0.f);
            if (t.k00) red_add(dxp, l00);
            if (t.k01 && !given) red_add(dxp + 1, t.w01 * g);
            if (t.k10) red_add(dxp + a.W, l10);
            if (t.k11 && !given) red_add(dxp + a.W + 1, t.w11 * g);
            dxp += HW;
        }
        gp += HW;
        xp += HW;
    }
    if (a.dflow && live) {
        float *dfp = a.dflow + (long long)n * 2 * HW + rem;
        dfp[0] = dix * cgx;
        dfp[HW] = diy * cgy;
    }
}

// ----------------------------------------------------------------- backward, warp windows
// d_input through a per-warp shared-memory window (the "bounded footprint" of the
// scatter, found at run time since a flow field has no inverse).
// The global reds are the limit of the per-tap kernel above: red.global issues at
// ~1.3 cycles per lane per SM, so ~3 reds per (pixel, channel) cost more than all
// other work.  Here a warp takes a 32-column strip of R consecutive rows; its taps
// are added (plain shared-memory read-modify-write, no atomics) into a window of
// kWinHS x kWinWU input pixels anchored at the strip's first-row floor cells, then
// the window is flushed with one red.global.add.v4.f32 per touched 16-B group:
// ~0.5 vector reds per (pixel, channel) for smooth flow instead of ~3 scalar reds.
// Lanes of one row instruction that share a floor cell (common for noisy flow) are
// first combined onto the lowest such lane by shuffles, so the read-modify-write of
// one instruction never has two lanes on the same address.  Taps whose cell falls
// outside the window (large or discontinuous flow) take direct reds.
constexpr int kWinHS = 16, kWinWU = 64, kWinRS = 68;  // rows, usable cols, row stride (floats)

// Per-row state of the software pipeline: the tap, this lane's dY and (for d_flow)
// X tap values of the current channel chunk, all loaded before the row is processed.
template <int CW>
struct WinRow {
    Tap t;
    float cgx, cgy;
    float g[CW];
    float v[CW][4];
};

template <int R, int NW, int CW>
__global__ void __launch_bounds__(NW * 32)
    warp_bwd_win(WarpArgs a, int tiles_x, int iters) {
    extern __shared__ __align__(16) float wsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = blockIdx.y;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int x = tx * 32 + lane;
    const bool xin = x < a.W;
    const int xs_ = xin ? x : 0;
    const int HW = a.H * a.W;
    constexpr int WF = kWinHS * kWinRS;  // floats per window channel
    float *win = wsm + w * CW * WF;
    for (int e = lane; e < CW * WF / 4; e += 32) ((float4 *)win)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    const bool vec = ((a.W & 3) == 0) && ((((uintptr_t)a.dx) & 15u) == 0);
    const bool need_df = a.dflow != nullptr;
    const float *fs = a.flow + (long long)n * 2 * HW;
    const int ybase = (ty * NW + w) * R * iters;

    for (int c0 = 0; c0 < a.C; c0 += CW) {
        const int cn = min(CW, a.C - c0);
        const float *xs = a.x + ((long long)n * a.C + c0) * HW;
        const float *gs = a.dy + ((long long)n * a.C + c0) * HW;
        float *dxs = a.dx + ((long long)n * a.C + c0) * HW;
        auto ld_flow = [&](int y, float &u, float &v) {
            u = v = 0.f;
            if (y < a.H && xin) {
                u = ldg_stream(fs + y * a.W + x);
                v = ldg_stream(fs + HW + y * a.W + x);
            }
        };
        // tap + dY + X loads of row y (all issued before any is consumed)
        auto mk_row = [&](int y, float u, float v, WinRow<CW> &r) {
            r.t = warp_tap(a, xs_, y, u, v, r.cgx, r.cgy);
            if (!xin || y >= a.H) r.t.k00 = r.t.k01 = r.t.k10 = r.t.k11 = false;
            const int rem = (y < a.H ? y : 0) * a.W + xs_;
            const int o = (int)r.t.o00;
#pragma unroll
            for (int c = 0; c < CW; c++) {
                r.g[c] = (c < cn && xin && y < a.H) ? ldg_stream(gs + (long long)c * HW + rem) : 0.f;
                const float *p = xs + (long long)c * HW + o;
                const bool lc = need_df && c < cn;
                r.v[c][0] = (lc && r.t.k00) ? TAPLD(p) : 0.f;
                r.v[c][1] = (lc && r.t.k01) ? TAPLD(p + 1) : 0.f;
                r.v[c][2] = (lc && r.t.k10) ? TAPLD(p + a.W) : 0.f;
                r.v[c][3] = (lc && r.t.k11) ? TAPLD(p + a.W + 1) : 0.f;
            }
        };
        for (int it = 0; it < iters; it++) {
            const int yr0 = ybase + it * R;
            if (yr0 >= a.H) break;
            float un, vn;
            ld_flow(yr0 + 1, un, vn);
            WinRow<CW> cur;
            {
                float u0, v0;
                ld_flow(yr0, u0, v0);
                mk_row(yr0, u0, v0, cur);
            }
            // window anchor: the strip's first-row floor cells
            const int gx0 = (__reduce_min_sync(0xffffffffu, xin ? cur.t.x0 : 0x3fffffff) - 12) & ~3;
            const int gy0 = __reduce_min_sync(0xffffffffu, xin ? cur.t.y0 : 0x3fffffff) - 4;
            int lxmin = 1 << 30, lxmax = -(1 << 30), lymin = 1 << 30, lymax = -(1 << 30);
#pragma unroll 1
            for (int rr = 0; rr < R; rr++) {
                const int y = yr0 + rr;
                if (y >= a.H) break;
                // pipeline: flow of row y+2 and taps / values of row y+1 in flight
                WinRow<CW> nxt;
                const bool more = rr + 1 < R && y + 1 < a.H;
                if (more) {
                    const float u1 = un, v1 = vn;
                    if (rr + 2 < R) ld_flow(y + 2, un, vn);
                    mk_row(y + 1, u1, v1, nxt);
                }
                const Tap &t = cur.t;
                const int lx = t.x0 - gx0, ly = t.y0 - gy0;
                const bool any = t.k00 || t.k01 || t.k10 || t.k11;
                const bool inwin = any && lx >= 0 && lx < kWinWU - 1 && ly >= 0 && ly < kWinHS - 1;
                const int key = inwin ? ly * kWinRS + lx : -1 - lane;
                const unsigned m = __match_any_sync(0xffffffffu, key);
                const bool leader = inwin && lane == __ffs(m) - 1;
                const int gsz = __reduce_max_sync(0xffffffffu, inwin ? __popc(m) : 1);
                if (inwin) {
                    lxmin = min(lxmin, lx);
                    lxmax = max(lxmax, lx);
                    lymin = min(lymin, ly);
                    lymax = max(lymax, ly);
                }
                if (need_df && xin) {
                    float dix = 0.f, diy = 0.f;
#pragma unroll
                    for (int c = 0; c < CW; c++) {
                        const float *vv = cur.v[c];
                        dix = fmaf(cur.g[c], fmaf(1.f - t.fy, vv[1] - vv[0], t.fy * (vv[3] - vv[2])), dix);
                        diy = fmaf(cur.g[c], fmaf(1.f - t.fx, vv[2] - vv[0], t.fx * (vv[3] - vv[1])), diy);
                    }
                    // C > CW: later chunks add onto the first chunk's value
                    float *dfp = a.dflow + (long long)n * 2 * HW + y * a.W + x;
                    if (c0 == 0) {
                        dfp[0] = dix * cur.cgx;
                        dfp[HW] = diy * cur.cgy;
                    } else {
                        dfp[0] += dix * cur.cgx;
                        dfp[HW] += diy * cur.cgy;
                    }
                }
                const unsigned m1 = m & (m - 1u);  // this lane's group without its leader
                const int src1 = m1 ? __ffs(m1) - 1 : lane;
                float *wrow = win + ly * kWinRS + lx;
#pragma unroll
                for (int c = 0; c < CW; c++) {
                    if (c >= cn) break;
                    const float g = cur.g[c];
                    const float v4[4] = {t.k00 ? t.w00 * g : 0.f, t.k01 ? t.w01 * g : 0.f,
                                         t.k10 ? t.w10 * g : 0.f, t.k11 ? t.w11 * g : 0.f};
                    float s4[4] = {v4[0], v4[1], v4[2], v4[3]};
                    if (gsz > 1) {
                        // the leader pulls its group's other members' own values
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            const float p1 = __shfl_sync(0xffffffffu, v4[k], src1);
                            if (src1 != lane) s4[k] += p1;
                        }
                        unsigned mr = m1 & (m1 - 1u);
                        for (int r = 2; r < gsz; r++, mr &= mr - 1u) {
                            const int sr = mr ? __ffs(mr) - 1 : lane;
#pragma unroll
                            for (int k = 0; k < 4; k++) {
                                const float pr = __shfl_sync(0xffffffffu, v4[k], sr);
                                if (sr != lane) s4[k] += pr;
                            }
                        }
                    }
                    // one tap kind at a time: a leader's right tap can be another
                    // leader's left tap, so the kinds are ordered by warp barriers
                    float *wp = wrow + c * WF;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        if (leader) wp[(k >> 1) * kWinRS + (k & 1)] += s4[k];
                        __syncwarp();
                    }
                    if (!inwin && any) {
                        float *dp = dxs + (long long)c * HW + (int)t.o00;
                        if (t.k00) red_add(dp, v4[0]);
                        if (t.k01) red_add(dp + 1, v4[1]);
                        if (t.k10) red_add(dp + a.W, v4[2]);
                        if (t.k11) red_add(dp + a.W + 1, v4[3]);
                    }
                }
                if (more) cur = nxt;
            }
            // flush the touched part of the window: one vector red per nonzero 16-B group
            lxmin = __reduce_min_sync(0xffffffffu, lxmin);
            lxmax = __reduce_max_sync(0xffffffffu, lxmax);
            lymin = __reduce_min_sync(0xffffffffu, lymin);
            lymax = __reduce_max_sync(0xffffffffu, lymax);
            if (lxmin <= lxmax) {
                const int q0 = lxmin >> 2, q1 = (lxmax + 1) >> 2, nq = q1 - q0 + 1;
                const int nr = lymax + 2 - lymin;
                const int tot = nq * nr * cn;
                for (int e = lane; e < tot; e += 32) {
                    const int c = e / (nq * nr), rem2 = e - c * nq * nr;
                    const int r = rem2 / nq, q = rem2 - r * nq;
                    float4 *wp = (float4 *)(win + c * WF + (lymin + r) * kWinRS) + q0 + q;
                    const float4 s = *wp;
                    if (s.x != 0.f || s.y != 0.f || s.z != 0.f || s.w != 0.f) {
                        *wp = make_float4(0.f, 0.f, 0.f, 0.f);
                        const int gy = gy0 + lymin + r, gx = gx0 + 4 * (q0 + q);
                        float *dp = dxs + (long long)c * HW + (long long)gy * a.W + gx;
                        if (vec) {
                            red_add_v4(dp, s.x, s.y, s.z, s.w);
                        } else {
                            const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
                            for (int k = 0; k < 4; k++)
                                if (sv[k] != 0.f && gx + k >= 0 && gx + k < a.W) red_add(dp + k, sv[k]);
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
}

}  // namespace

size_t warp_ws_bytes(int N, int C, int H, int W) {
    (void)N;
    (void)C;
    (void)H;
    (void)W;
    return 0;
}

// Optional tiled path (RSGRAD_WARP=tiled): the staged-footprint output-tile kernel of
// stn.cu with flow coordinates.  Measured slower than the per-pixel kernels below at
// C = 3 (fwd 0.41 vs 0.29 ms, bwd 0.74 vs 0.62 ms at 16x3x1024^2): the footprint setup
// is amortised over too few channels, so the direct kernels are the default.
static StnArgs as_tile_args(const WarpArgs &a) {
    StnArgs t{};
    t.x = a.x; t.dy = a.dy; t.y = a.y; t.dx = a.dx;
    t.N = a.N; t.C = a.C; t.H = a.H; t.W = a.W; t.Ho = a.H; t.Wo = a.W;
    t.ac = 1; t.border = a.border;
    t.flow = a.flow; t.dflow = a.dflow;
    return t;
}

static bool warp_direct() {
    const char *e = getenv("RSGRAD_WARP");
    return !(e && strcmp(e, "tiled") == 0);
}

cudaError_t warp_fwd_launch(const WarpArgs &a, cudaStream_t s) {
    if (!warp_direct()) return flow_tile_launch(as_tile_args(a), 0, false, s);
    const int HW = a.H * a.W;
    warp_fwd_kernel<<<dim3((HW + kThreads - 1) / kThreads, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
    note_launch();
    return cudaGetLastError();
}

cudaError_t warp_bwd_launch(const WarpArgs &a, int algo, int deterministic, void *ws,
                            size_t ws_bytes, cudaStream_t s) {
    (void)deterministic;
    (void)ws;
    (void)ws_bytes;
    const long long HW = (long long)a.H * a.W;
    if (a.dx) {
        cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * HW, s);
        if (e != cudaSuccess) return e;
    }
    // SCATTER_PRIV: d_input through a block-private footprint accumulator (one red per
    // touched input element per tile) instead of per-tap global reds
    if (algo == 2 || !warp_direct()) return flow_tile_launch(as_tile_args(a), 2, algo == 2, s);
    // AUTO / SCATTER_ATOMIC: per-tap reds (warp_bwd_kernel).  RSGRAD_WARP_BWD=winR,NW,IT
    // selects the per-warp shared windows flushed by vector reds (warp_bwd_win): 2.5x
    // less L2 traffic, but measured slower at configs[4] (0.65 vs 0.59 ms at 16 x 3 x
    // 1024^2): the per-tap kernel is bound by L1 (83%, the d_flow tap gathers as much
    // as the reds), the window kernel by shared-memory latency at 22% occupancy.
    const char *e = getenv("RSGRAD_WARP_BWD");
    const bool direct = algo == 3 || !a.dx || !(e && strncmp(e, "win", 3) == 0);
    if (direct) {
        warp_bwd_kernel<<<dim3((unsigned)((HW + kThreads - 1) / kThreads), a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
        note_launch();
        return cudaGetLastError();
    }
    int R = 8, NW = 4, iters = 4;
    if (e && strncmp(e, "win", 3) == 0) sscanf(e + 3, "%d,%d,%d", &R, &NW, &iters);
    const int CW = a.C < 3 ? a.C : 3;
    const int tiles_x = (a.W + 31) / 32, rows = R * NW * iters;
    const int tiles_y = (a.H + rows - 1) / rows;
    const size_t sm = sizeof(float) * (size_t)NW * CW * kWinHS * kWinRS;
    const dim3 grid((unsigned)(tiles_x * tiles_y), a.N);
    auto go = [&](auto kern) {
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<grid, NW * 32, sm, s>>>(a, tiles_x, iters);
    };
#define RS_WIN(RR, NN)                                                      \
    if (R == RR && NW == NN) {                                              \
        if (CW == 1) go(warp_bwd_win<RR, NN, 1>);                           \
        else if (CW == 2) go(warp_bwd_win<RR, NN, 2>);                      \
        else go(warp_bwd_win<RR, NN, 3>);                                   \
    } else
    RS_WIN(8, 4) RS_WIN(4, 8) RS_WIN(8, 8) RS_WIN(4, 4) { return cudaErrorInvalidValue; }
#undef RS_WIN
    note_launch();
    return cudaGetLastError();
}

}  // namespace rs
