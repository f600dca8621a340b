// warp.cu — FlowNet 2.0 per-pixel warp, forward and adjoint, sm_100a.
//
// Kernels
//   warp_fwd_px<2>    two pixels per thread (loads of both issued first): coordinate
//                     x + u(x) in fp64, bilinear gather over all channels
//                     (warp_fwd_kernel: one pixel per thread, RSGRAD_WARP_FWD_PX=1).
//   warp_bwd_kernel   one thread per pixel: d_flow is a pure gather (G and the X
//                     taps); d_input is the reversed gather, which for an
//                     arbitrary flow field has no bounded inverse, so it is
//                     "a general scatter using atomics": fp32
//                     red.global.add into a zero-filled dx (AUTO, SCATTER_ATOMIC).
//   warp_bwd_win      variant (RSGRAD_WARP_BWD=winR,NW,IT): per-warp shared windows
//                     flushed by red.v4 (measured slower).
//   SCATTER_PRIV goes through the staged-footprint output tile of stn.cu (flow mode).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "det.cuh"

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

// One group of PX pixels per thread (base + k * kThreads, k < PX) of sample n, flow values
// already loaded: every tap load of a channel for all PX pixels is issued before its
// first use (memory-level parallelism for the latency-bound gather).
template <int PX>
RS_DEV void warp_fwd_group(const WarpArgs &a, double invW, int n, int base, const float *u, const float *v) {
    const int HW = a.H * a.W;
    int o[PX];
    float w[PX][4];
#pragma unroll
    for (int k = 0; k < PX; k++) {
        const int rem = base + k * kThreads;
        const int rc = min(rem, HW - 1);
        const int y = fast_div(rc, a.W, invW), x = rc - y * a.W;
        float cgx, cgy;
        const Tap t = warp_tap(a, x, y, u[k], v[k], cgx, cgy);
        const bool live = rem < HW;
        // cell fully inside: 4 unconditional taps; a cell at the image edge (some taps
        // outside) takes the exact per-tap gather below (o = -1); else no taps (o = -2)
        const bool full = t.k00 && t.k01 && t.k10 && t.k11;
        o[k] = !live ? -2 : full ? (int)t.o00 : (t.k00 || t.k01 || t.k10 || t.k11) ? -1 : -2;
        w[k][0] = t.w00;
        w[k][1] = t.w01;
        w[k][2] = t.w10;
        w[k][3] = t.w11;
    }
    const float *xp = a.x + (long long)n * a.C * HW;
    float *yp = a.y + (long long)n * a.C * HW;
    for (int c = 0; c < a.C; c++) {
        float r[PX];
#pragma unroll
        for (int k = 0; k < PX; k++) {
            if (o[k] >= 0) {
                const float *p = xp + o[k];
                const float t0 = TAPLD(p), t1 = TAPLD(p + 1), t2 = TAPLD(p + a.W), t3 = TAPLD(p + a.W + 1);
                r[k] = fmaf(w[k][3], t3, fmaf(w[k][2], t2, fmaf(w[k][1], t1, fmaf(w[k][0], t0, 0.f))));
            } else {
                r[k] = 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < PX; k++) {
            const int rem = base + k * kThreads;
            if (rem >= HW) continue;
            if (o[k] == -1) {  // edge cell: the exact per-tap gather of warp_fwd_kernel
                const int y = fast_div(rem, a.W, invW), x = rem - y * a.W;
                float cgx, cgy;
                const Tap t = warp_tap(a, x, y, u[k], v[k], cgx, cgy);
                const float *p = xp + t.o00;
                float q = 0.f;
                if (t.k00) q = fmaf(t.w00, TAPLD(p), q);
                if (t.k01) q = fmaf(t.w01, TAPLD(p + 1), q);
                if (t.k10) q = fmaf(t.w10, TAPLD(p + a.W), q);
                if (t.k11) q = fmaf(t.w11, TAPLD(p + a.W + 1), q);
                r[k] = q;
            }
            yp[rem] = r[k];
        }
        xp += HW;
        yp += HW;
    }
}

// PX pixels per thread, one group per thread
template <int PX>
__global__ void __launch_bounds__(kThreads) warp_fwd_px(WarpArgs a, double invW) {
    const int HW = a.H * a.W;
    const int base = blockIdx.x * kThreads * PX + threadIdx.x;
    const int n = blockIdx.y;
    const float *fp = a.flow + (long long)n * 2 * HW;
    float u[PX], v[PX];
#pragma unroll
    for (int k = 0; k < PX; k++) {
        const int rem = min(base + k * kThreads, HW - 1);
        u[k] = ldg_stream(fp + rem);
        v[k] = ldg_stream(fp + HW + rem);
    }
    warp_fwd_group<PX>(a, invW, n, base, u, v);
}

// G consecutive groups of PX pixels per thread; the next group's flow loads are issued
// before the current group's taps (the flow -> coordinate -> tap dependency otherwise
// exposes one full memory round trip per group)
template <int PX, int G>
__global__ void __launch_bounds__(kThreads) warp_fwd_pipe(WarpArgs a, double invW) {
    const int HW = a.H * a.W;
    const int per = kThreads * PX;
    const int b0 = blockIdx.x * per * G;
    const int n = blockIdx.y;
    const float *fp = a.flow + (long long)n * 2 * HW;
    float un[PX], vn[PX];
    auto fetch = [&](int g) {
#pragma unroll
        for (int k = 0; k < PX; k++) {
            const int rem = min(b0 + g * per + k * kThreads + (int)threadIdx.x, HW - 1);
            un[k] = ldg_stream(fp + rem);
            vn[k] = ldg_stream(fp + HW + rem);
        }
    };
    fetch(0);
#pragma unroll 1
    for (int g = 0; g < G; g++) {
        if (b0 + g * per >= HW) break;  // block-uniform
        float u[PX], v[PX];
#pragma unroll
        for (int k = 0; k < PX; k++) { u[k] = un[k]; v[k] = vn[k]; }
        if (g + 1 < G) fetch(g + 1);
        warp_fwd_group<PX>(a, invW, n, b0 + g * per + (int)threadIdx.x, u, v);
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

// ----------------------------------------------------------------- backward, row strips (AUTO)
// d_input as a scatter whose overlapping writes are combined in registers before they
// reach memory (PAPER.md:733's atomics, applied to pre-summed values).  Lane = column
// x, a warp walks R consecutive rows of its 32 columns, block = kStripW warps stacked
// vertically.  Each lane keeps the 4 tap sums of its CURRENT floor cell pending:
//   * next row's cell == the same cell (vertical compression): add into the pending sums;
//   * next row's cell == the cell one row down (the common, smooth case): the pending
//     lower taps ARE the new cell's upper taps -- carried, only the upper pair is emitted;
//   * otherwise: all 4 pending sums are emitted.
// Emitted sums of lanes that share an element are merged across lanes before the red:
// a lane whose left taps are its left neighbour's right taps absorbs them (one shuffle
// per tap), and runs of lanes on the SAME cell (horizontal compression) are summed by
// a segmented shuffle scan onto the run's first lane.  Smooth flow: ~1 red per
// (pixel, channel) instead of ~2.2; a collapsing flow: the red count per element drops
// by the compression in both axes, which is also what keeps the fp32 reds' rounding
// (sequential in the order the L2 applies them) inside the tolerance.
// d_flow is the gather of the same pass; the X taps of a cell one row down reuse the
// two lower tap values already loaded.
#ifndef RS_STRIP_W
#define RS_STRIP_W 1
#endif
constexpr int kStripW = RS_STRIP_W;  // warps per block (1 measured best: configs[2] smooth 62.5 vs 68.6 us with 4)

#ifndef RS_STRIP_MINB
#define RS_STRIP_MINB (24 / RS_STRIP_W)  // 80 registers
#endif
// A run of lanes whose pre-summed emission carries >= kHeavyFanin taps marks the sample
// "heavy" (heavy[n] = this call's tag): a flow that folds that many pixels onto one cell puts hundreds
// of taps on an element, where even pre-summed fp32 partials round at the 1e-6 level of
// T's absolute floor; the launcher then recomputes that sample's d_input with the
// fixed-point scatter (det.cuh), exact to ~1e-11.  Smooth flows never get there (runs of
// <= 3 lanes, a row or two per cell).
constexpr int kHeavyFanin = 32;

template <int CW, int R>
__global__ void __launch_bounds__(kStripW * 32, RS_STRIP_MINB)
    warp_bwd_strip(WarpArgs a, int tiles_x, int *__restrict__ heavy, int tag, unsigned *__restrict__ det_zero = nullptr,
                   int nzero = 0) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = blockIdx.y;
    // the heavy-sample recompute's barrier / max slots, zeroed here instead of by a
    // separate memset on the stream (the recompute kernel runs after this one)
    if (det_zero && blockIdx.x == 0 && blockIdx.y == 0)
        for (int e = threadIdx.x; e < nzero; e += blockDim.x) det_zero[e] = 0u;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int x = tx * 32 + lane;
    const bool xin = x < a.W;
    const int HW = a.H * a.W;
    const int ybeg = (ty * kStripW + w) * R;
    if (ybeg >= a.H) return;  // warp-uniform
    const int yend = min(a.H, ybeg + R);
    const float *fs = a.flow + (long long)n * 2 * HW;
    const bool need_df = a.dflow != nullptr, need_dx = a.dx != nullptr;

    for (int c0 = 0; c0 < a.C; c0 += CW) {
        const int cn = min(CW, a.C - c0);
        const float *xs = a.x + ((long long)n * a.C + c0) * HW;
        const float *gs = a.dy + ((long long)n * a.C + c0) * HW;
        float *dxs = need_dx ? a.dx + ((long long)n * a.C + c0) * HW : nullptr;
        // pending cell of this lane
        bool have = false;
        int pcx = 0, pcy = 0, cnt = 0;  // pending cell; cnt: rows pre-summed into it
        bool pk[4] = {false, false, false, false};
        float pend[CW][4], xv[CW][4];
#pragma unroll
        for (int c = 0; c < CW; c++)
#pragma unroll
            for (int k = 0; k < 4; k++) pend[c][k] = xv[c][k] = 0.f;

        // Emit the pending sums selected by em[] (warp-collective: every lane calls it).
        auto emit = [&](bool e00, bool e01, bool e10, bool e11) {
            bool em[4] = {e00 && pk[0], e01 && pk[1], e10 && pk[2], e11 && pk[3]};
            const bool any = em[0] || em[1] || em[2] || em[3];
            const unsigned emk = (unsigned)em[0] | ((unsigned)em[1] << 1) | ((unsigned)em[2] << 2) |
                                 ((unsigned)em[3] << 3);
            // runs of lanes emitting the same set on the same cell
            const int ppx = __shfl_up_sync(0xffffffffu, pcx, 1), ppy = __shfl_up_sync(0xffffffffu, pcy, 1);
            const unsigned pem = __shfl_up_sync(0xffffffffu, emk, 1);
            const bool same_prev0 = lane > 0 && any && pem == emk && ppx == pcx && ppy == pcy;
            const unsigned runs0 = __ballot_sync(0xffffffffu, same_prev0);
            // combine only where it matters for the rounding: a run of >= 3 lanes on one
            // cell somewhere in the warp (pairs of jittered samples just red twice)
            const bool scan = (runs0 & (runs0 << 1)) != 0u;
            const bool same_prev = scan && same_prev0;
            const unsigned runs = scan ? runs0 : 0u;
            float val[CW][4];
#pragma unroll
            for (int c = 0; c < CW; c++)
#pragma unroll
                for (int k = 0; k < 4; k++) val[c][k] = pend[c][k];
            if (runs) {
                // segmented suffix sum: every run's first lane gets the run total
                const unsigned heads = ~runs;  // bit l: lane l starts a run (or is alone)
                const unsigned after = (lane == 31) ? 0u : (heads >> (lane + 1)) << (lane + 1);
                const int seg_end = after ? __ffs(after) - 2 : 31;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                    for (int c = 0; c < CW; c++)
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            const float t = __shfl_down_sync(0xffffffffu, val[c][k], o);
                            if (lane + o <= seg_end) val[c][k] += t;
                        }
                }
                if (heavy) {  // taps pre-summed by the run's first lane
                    int tot = any ? cnt : 0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t2 = __shfl_down_sync(0xffffffffu, tot, o);
                        if (lane + o <= seg_end) tot += t2;
                    }
                    if (__ballot_sync(0xffffffffu, !same_prev && tot >= kHeavyFanin) && lane == 0) heavy[n] = tag;
                }
                if (same_prev) em[0] = em[1] = em[2] = em[3] = false;
            }
            // the previous emitter's right taps on our left taps (same cell row, one column
            // left): the previous emitter is the head of the previous run (the left
            // neighbour lane when there are no runs), the next one takes ours
            const unsigned heads = runs ? ~runs : 0xffffffffu;
            const unsigned below = heads & ((1u << lane) - 1u);
            const int prevh = below ? 31 - __clz(below) : lane;
            const unsigned above = lane == 31 ? 0u : (heads & (~0u << (lane + 1)));
            const int nexth = above ? __ffs(above) - 1 : lane;
            const int qpx = __shfl_sync(0xffffffffu, pcx, prevh), qpy = __shfl_sync(0xffffffffu, pcy, prevh);
            const bool p01 = __shfl_sync(0xffffffffu, (int)em[1], prevh) != 0;
            const bool p11 = __shfl_sync(0xffffffffu, (int)em[3], prevh) != 0;
            const bool adj = prevh != lane && qpx + 1 == pcx && qpy == pcy;
            const bool ab01 = adj && p01 && em[0], ab11 = adj && p11 && em[2];
            const bool g01 = __shfl_sync(0xffffffffu, (int)ab01, nexth) != 0 && nexth != lane;
            const bool g11 = __shfl_sync(0xffffffffu, (int)ab11, nexth) != 0 && nexth != lane;
            if (g01) em[1] = false;
            if (g11) em[3] = false;
            const int o00 = any ? pcy * a.W + pcx : 0;  // a tap of the cell is in the image
#pragma unroll
            for (int c = 0; c < CW; c++) {
                const float r01 = __shfl_sync(0xffffffffu, val[c][1], prevh);
                const float r11 = __shfl_sync(0xffffffffu, val[c][3], prevh);
                if (c >= cn) continue;
                float *dp = dxs + (long long)c * HW + o00;
                const float v00 = val[c][0] + (ab01 ? r01 : 0.f), v10 = val[c][2] + (ab11 ? r11 : 0.f);
                if (em[0] && v00 != 0.f) red_add(dp, v00);
                if (em[1] && val[c][1] != 0.f) red_add(dp + 1, val[c][1]);
                if (em[2] && v10 != 0.f) red_add(dp + a.W, v10);
                if (em[3] && val[c][3] != 0.f) red_add(dp + a.W + 1, val[c][3]);
            }
        };

        float un = 0.f, vn = 0.f, gn[CW];
#pragma unroll
        for (int c = 0; c < CW; c++) gn[c] = 0.f;
        if (xin) {
            un = ldg_stream(fs + ybeg * a.W + x);
            vn = ldg_stream(fs + HW + ybeg * a.W + x);
#pragma unroll
            for (int c = 0; c < CW; c++)
                if (c < cn) gn[c] = ldg_stream(gs + (long long)c * HW + ybeg * a.W + x);
        }
#pragma unroll 1
        for (int y = ybeg; y < yend; y++) {
            const float u = un, v = vn;
            float g[CW];
#pragma unroll
            for (int c = 0; c < CW; c++) g[c] = gn[c];
            if (xin && y + 1 < yend) {  // prefetch the next row's flow and dY
                un = ldg_stream(fs + (y + 1) * a.W + x);
                vn = ldg_stream(fs + HW + (y + 1) * a.W + x);
#pragma unroll
                for (int c = 0; c < CW; c++)
                    if (c < cn) gn[c] = ldg_stream(gs + (long long)c * HW + (y + 1) * a.W + x);
            }
            float cgx, cgy;
            Tap t = warp_tap(a, xin ? x : 0, y, u, v, cgx, cgy);
            if (!xin) t.k00 = t.k01 = t.k10 = t.k11 = false;
            const bool tany = t.k00 || t.k01 || t.k10 || t.k11;
            const int rem = y * a.W + (xin ? x : 0);
            // relation of this row's cell to the pending one
            const bool same = have && t.x0 == pcx && t.y0 == pcy;
            const bool down = have && t.x0 == pcx && t.y0 == pcy + 1;
            if (need_df) {
                const int o = (int)t.o00;
#pragma unroll
                for (int c = 0; c < CW; c++) {
                    if (c >= cn) break;
                    const float *p = xs + (long long)c * HW + o;
                    if (!same) {
                        if (down) {
                            xv[c][0] = xv[c][2];
                            xv[c][1] = xv[c][3];
                        } else {
                            xv[c][0] = t.k00 ? TAPLD(p) : 0.f;
                            xv[c][1] = t.k01 ? TAPLD(p + 1) : 0.f;
                        }
                        xv[c][2] = t.k10 ? TAPLD(p + a.W) : 0.f;
                        xv[c][3] = t.k11 ? TAPLD(p + a.W + 1) : 0.f;
                    }
                }
                float dix = 0.f, diy = 0.f;
#pragma unroll
                for (int c = 0; c < CW; c++) {
                    if (c >= cn) break;
                    dix = fmaf(g[c], fmaf(1.f - t.fy, xv[c][1] - xv[c][0], t.fy * (xv[c][3] - xv[c][2])), dix);
                    diy = fmaf(g[c], fmaf(1.f - t.fx, xv[c][2] - xv[c][0], t.fx * (xv[c][3] - xv[c][1])), diy);
                }
                if (xin) {
                    float *dfp = a.dflow + (long long)n * 2 * HW + rem;
                    if (c0 == 0) {
                        dfp[0] = dix * cgx;
                        dfp[HW] = diy * cgy;
                    } else {  // C > CW: later chunks add onto the first chunk's value
                        dfp[0] += dix * cgx;
                        dfp[HW] += diy * cgy;
                    }
                }
            }
            if (need_dx) {
                // emit what this row does not continue (warp-collective)
                const bool keep_all = same || (!have);
                emit(!keep_all, !keep_all, !keep_all && !down, !keep_all && !down);
                float nv[CW][4];
#pragma unroll
                for (int c = 0; c < CW; c++) {
                    nv[c][0] = t.w00 * g[c];
                    nv[c][1] = t.w01 * g[c];
                    nv[c][2] = t.w10 * g[c];
                    nv[c][3] = t.w11 * g[c];
                }
                if (same) {
#pragma unroll
                    for (int c = 0; c < CW; c++)
#pragma unroll
                        for (int k = 0; k < 4; k++) pend[c][k] += nv[c][k];
                } else if (down) {
#pragma unroll
                    for (int c = 0; c < CW; c++) {
                        pend[c][0] = pend[c][2] + nv[c][0];
                        pend[c][1] = pend[c][3] + nv[c][1];
                        pend[c][2] = nv[c][2];
                        pend[c][3] = nv[c][3];
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < CW; c++)
#pragma unroll
                        for (int k = 0; k < 4; k++) pend[c][k] = nv[c][k];
                }
                cnt = (same || down) ? cnt + 1 : 1;
                have = tany;
                pcx = t.x0;
                pcy = t.y0;
                pk[0] = t.k00;
                pk[1] = t.k01;
                pk[2] = t.k10;
                pk[3] = t.k11;
            } else {
                have = tany;
                pcx = t.x0;
                pcy = t.y0;
            }
        }
        if (need_dx) emit(true, true, true, true);
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

// Warp taps for the deterministic fixed-point scatter (det.cuh): the coordinate and
// weights of warp_tap.
struct WarpTapSampler {
    WarpArgs a;
    static constexpr int kMaxTaps = 4;
    static constexpr double kWmax = 1.0;
    RS_DEV int taps(int n, long long q, long long *off, float *w) const {
        const int HW = a.H * a.W;
        const int y = (int)(q / a.W), x = (int)(q - (long long)y * a.W);
        const float *fp = a.flow + (long long)n * 2 * HW + q;
        float cgx, cgy;
        const Tap t = warp_tap(a, x, y, __ldg(fp), __ldg(fp + HW), cgx, cgy);
        int k = 0;
        if (t.k00) { off[k] = t.o00; w[k++] = t.w00; }
        if (t.k01) { off[k] = t.o00 + 1; w[k++] = t.w01; }
        if (t.k10) { off[k] = t.o00 + a.W; w[k++] = t.w10; }
        if (t.k11) { off[k] = t.o00 + a.W + 1; w[k++] = t.w11; }
        return k;
    }
};

}  // namespace

// AUTO and deterministic=1 both may run the fixed-point scatter (AUTO: for samples the
// strip kernel marks heavy); AUTO also keeps the per-sample heavy flags after it
size_t warp_ws_bytes(int N, int C, int H, int W, bool det) {
    return det_align(det_ws_bytes(N, (long long)C * H * W)) + (det ? 0 : det_align(sizeof(int) * (size_t)N));
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
    static const int px = [] {
        const char *e = getenv("RSGRAD_WARP_FWD_PX");
        return e ? atoi(e) : 2;  // 2 px per thread: 0.703 vs 0.768 ms at 64 x 1024^2 (4: 1.01)
    }();
    // four pixel pairs per thread with the flow of the next pair prefetched (0.70 -> 0.64 ms
    // at 64 x 1024^2) when the grid stays many waves deep; small batches keep one pair per
    // thread (configs[2]: 26.6 vs 32.8 us with four -- a quarter of the blocks)
    const char *eg = getenv("RSGRAD_WARP_FWD_G");  // (read per call: tests switch it)
    const int groups = eg ? atoi(eg) : ((long long)a.N * HW >= (16LL << 20) ? 4 : 1);
    if (px == 2 && groups == 4) {
        const int per = kThreads * 2 * 4;
        warp_fwd_pipe<2, 4><<<dim3((HW + per - 1) / per, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
    } else if (px == 2 && groups == 2) {
        const int per = kThreads * 2 * 2;
        warp_fwd_pipe<2, 2><<<dim3((HW + per - 1) / per, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
    } else if (px == 2 || px == 4) {
        const int per = kThreads * px;
        if (px == 2) warp_fwd_px<2><<<dim3((HW + per - 1) / per, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
        else warp_fwd_px<4><<<dim3((HW + per - 1) / per, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
    } else {
        warp_fwd_kernel<<<dim3((HW + kThreads - 1) / kThreads, a.N), kThreads, 0, s>>>(a, 1.0 / a.W);
    }
    note_launch();
    return cudaGetLastError();
}

cudaError_t warp_bwd_launch(const WarpArgs &a, int algo, int deterministic, void *ws,
                            size_t ws_bytes, cudaStream_t s) {
    (void)ws_bytes;
    const long long HW = (long long)a.H * a.W;
    if (deterministic && a.dx) {
        // deterministic=1: d_flow by the strip kernel's gather alone, d_input by the
        // fixed-point scatter (bitwise reproducible, det.cuh)
        if (a.dflow) {
            WarpArgs b = a;
            b.dx = nullptr;
            cudaError_t e = warp_bwd_launch(b, 0, 0, nullptr, 0, s);
            if (e != cudaSuccess) return e;
        }
        return det_scatter_launch(WarpTapSampler{a}, a.dy, a.dx, a.N, a.C, HW, HW, nullptr, nullptr, nullptr, ws, s);
    }
    if (a.dx) {
        cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * HW, s);
        if (e != cudaSuccess) return e;
    }
    // SCATTER_PRIV: d_input through a block-private footprint accumulator (one red per
    // touched input element per tile) instead of per-tap global reds
    if (algo == 2 || !warp_direct()) return flow_tile_launch(as_tile_args(a), 2, algo == 2, s);
    // AUTO: row strips with register-combined taps (warp_bwd_strip).  SCATTER_ATOMIC:
    // one red per tap (warp_bwd_kernel, the unconverted scatter).  RSGRAD_WARP_BWD=winR,NW,IT
    // selects the per-warp shared windows flushed by vector reds (warp_bwd_win),
    // RSGRAD_WARP_BWD=direct the per-tap kernel (A/B measurements).
    const char *e = getenv("RSGRAD_WARP_BWD");
    const bool win = algo != 3 && a.dx && e && strncmp(e, "win", 3) == 0;
    const bool direct = algo == 3 || (e && strcmp(e, "direct") == 0);
    if (!win && !direct) {
        const int tiles_x = (a.W + 31) / 32;
        // rows per warp: 8 (measured vs 16: 523 vs 536 us at 16 x 3 x 1024^2).  Not fewer: the
        // rows a lane walks are also what pre-sums a vertically collapsing flow's taps
        // before the reds (R = 4 let the 8 x 3 x 384 x 512 collapse test exceed T once)
        int R = 8;
        const char *er = getenv("RSGRAD_WARP_R");
        if (er) R = atoi(er) == 16 ? 16 : 8;
        const int tiles_y = (a.H + R * kStripW - 1) / (R * kStripW);
        const dim3 grid((unsigned)(tiles_x * tiles_y), a.N);
        const int CW = a.C < 4 ? a.C : 4;
        // heavy-sample flags (d_input only; none when the workspace cannot hold the fixed point)
        const bool rescue = a.dx && ws && ws_bytes >= warp_ws_bytes(a.N, a.C, a.H, a.W, false);
        int *heavy = rescue ? (int *)((char *)ws + det_align(det_ws_bytes(a.N, (long long)a.C * HW))) : nullptr;
        unsigned *dz = rescue ? det_ws_layout(ws, a.N, (long long)a.C * HW).bar : nullptr;
        const int nz = a.N + 2;
        // a fresh tag per call instead of clearing the flags (a stale match in reused memory
        // would only send that sample through the exact recompute)
        static std::atomic<unsigned> tags{0};
        const int tag = (int)(tags.fetch_add(1u) % 0x7ffffff0u) + 2;
#define RS_STRIP(RR)                                                                                        \
    switch (CW) {                                                                                           \
        case 1: warp_bwd_strip<1, RR><<<grid, kStripW * 32, 0, s>>>(a, tiles_x, heavy, tag, dz, nz); break;              \
        case 2: warp_bwd_strip<2, RR><<<grid, kStripW * 32, 0, s>>>(a, tiles_x, heavy, tag, dz, nz); break;              \
        case 3: warp_bwd_strip<3, RR><<<grid, kStripW * 32, 0, s>>>(a, tiles_x, heavy, tag, dz, nz); break;              \
        default: warp_bwd_strip<4, RR><<<grid, kStripW * 32, 0, s>>>(a, tiles_x, heavy, tag, dz, nz); break;             \
    }
        if (R == 8) {
            RS_STRIP(8)
        } else {
            RS_STRIP(16)
        }
#undef RS_STRIP
        note_launch();
        if (heavy) {  // heavy samples only (the others exit at once): d_input in fixed point
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            // (slots zeroed by the strip kernel; one block per SM: the grid mostly exits at once)
            return det_scatter_launch(WarpTapSampler{a}, a.dy, a.dx, a.N, a.C, HW, HW, nullptr, nullptr, heavy, ws, s,
                                      tag, false, 1);
        }
        return cudaGetLastError();
    }
    if (direct || !win) {
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
