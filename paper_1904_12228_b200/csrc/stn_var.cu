// stn_var.cu — STN variants the paper names (PAPER.md:28:
// "changing the interpolation scheme ... or interpolating over more dimensions"), sm_100a.
//
//   bicubic STN   Keys' cubic convolution (A = -0.75) over the 4 x 4 taps around the
//                 affine sample point, zeros outside (R12).
//   3-D STN       volumetric affine_grid (theta 3 x 4) + trilinear sampling.
// Coordinates are evaluated in fp64 in the oracle's order (P1); tap weights and their
// derivatives in fp64, rounded to fp32 for the per-channel data arithmetic.
// Forward: thread per output pixel, taps through L1.  Adjoint: d_theta per pixel ->
// warp -> block (fp32) -> fp64 block partials -> fixed-order sum; d_input of the bicubic
// STN by the converted gather over the affine preimage (bicubic_dx_gather: GATHER or
// deterministic=1) or the general scatter with atomics (AUTO / SCATTER_ATOMIC, and the 3-D
// STN: PAPER.md:733's fallback).
#include "common.cuh"
#include "det.cuh"

namespace rs {
namespace {

constexpr int kVT = 256;

// Output pixel of this thread.  When the output tiles exactly into 32 x 8 blocks, each
// warp covers a 16 x 2 patch: under a rotation the 32 lanes of one tap load then touch
// fewer input rows than a 32-pixel row run (up to 16 rows at 30 degrees), so each load
// costs fewer L1 wavefronts (measured: 16 x 2 < 8 x 4 < 4 x 8 in time).  Otherwise (ragged shapes) row-major runs of 256.  Either way a block owns
// 256 output pixels and the grid has P / 256 blocks per sample (d_theta partial slots).
#ifndef RS_PATCH_W
#define RS_PATCH_W 16
#endif
RS_DEV int out_pixel(int Ho, int Wo) {
    if ((Wo & 31) == 0 && (Ho & 7) == 0) {
        const int tw = Wo >> 5, ty = blockIdx.x / tw, tx = blockIdx.x - ty * tw;
        constexpr int PW = RS_PATCH_W, PH = 32 / PW, WA = 32 / PW;  // warp patch PW x PH
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        return (ty * 8 + (w / WA) * PH + l / PW) * Wo + tx * 32 + (w % WA) * PW + l % PW;
    }
    return blockIdx.x * kVT + threadIdx.x;
}

RS_DEV void cubic_w(double t, float w[4], float dw[4]) {
    const double A = -0.75;
    auto c1 = [&](double x) { return __dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn(__dmul_rn(A + 2.0, x), A + 3.0), x), x), 1.0); };
    auto c2 = [&](double x) {
        return __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(A, x), 5.0 * A), x), 8.0 * A), x), 4.0 * A);
    };
    auto d1 = [&](double x) { return __dmul_rn(__dsub_rn(__dmul_rn(3.0 * (A + 2.0), x), 2.0 * (A + 3.0)), x); };
    auto d2 = [&](double x) { return __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(3.0 * A, x), 10.0 * A), x), 8.0 * A); };
    w[0] = (float)c2(t + 1.0);
    w[1] = (float)c1(t);
    w[2] = (float)c1(1.0 - t);
    w[3] = (float)c2(2.0 - t);
    dw[0] = (float)d2(t + 1.0);
    dw[1] = (float)d1(t);
    dw[2] = (float)-d1(1.0 - t);
    dw[3] = (float)-d2(2.0 - t);
}

struct Bicubic {
    int x0, y0;  // floor of the sample point
    float wx[4], wy[4], dwx[4], dwy[4];
    double xt, yt;
};

RS_DEV Bicubic bicubic_at(const float *theta, int n, int i, int j, int H, int W, int Ho, int Wo, int ac) {
    Bicubic b;
    b.xt = stn_norm(j, Wo, ac);
    b.yt = stn_norm(i, Ho, ac);
    const float *t = theta + 6 * n;
    const double ix = stn_unnorm(affine3(__ldg(t), __ldg(t + 1), __ldg(t + 2), b.xt, b.yt), W, ac);
    const double iy = stn_unnorm(affine3(__ldg(t + 3), __ldg(t + 4), __ldg(t + 5), b.xt, b.yt), H, ac);
    const Cell cx = cell_of(ix), cy = cell_of(iy);
    b.x0 = cx.i0;
    b.y0 = cy.i0;
    cubic_w(__dsub_rn(ix, floor(ix)), b.wx, b.dwx);
    cubic_w(__dsub_rn(iy, floor(iy)), b.wy, b.dwy);
    return b;
}

__global__ void __launch_bounds__(kVT) bicubic_fwd(StnArgs a) {
    const int P = a.Ho * a.Wo, HW = a.H * a.W;
    const int q = out_pixel(a.Ho, a.Wo);
    if (q >= P) return;
    const int n = blockIdx.y, i = q / a.Wo, j = q - i * a.Wo;
    const Bicubic b = bicubic_at(a.theta, n, i, j, a.H, a.W, a.Ho, a.Wo, a.ac);
    for (int c = 0; c < a.C; c++) {
        const float *p = a.x + ((long long)n * a.C + c) * HW;
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int yy = b.y0 - 1 + u;
            if (yy < 0 || yy >= a.H) continue;
            float r = 0.f;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const int xx = b.x0 - 1 + v;
                if (xx >= 0 && xx < a.W) r = fmaf(b.wx[v], __ldg(p + yy * a.W + xx), r);
            }
            s = fmaf(b.wy[u], r, s);
        }
        a.y[((long long)n * a.C + c) * P + q] = s;
    }
}

// block reduction of NV fp32 values into fp64 partial slot `out` (thread 0 writes)
template <int NV>
RS_DEV void block_partial(float (&v)[NV], double *out) {
    __shared__ float red[kVT / 32][NV];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const float s = warp_sum(v[k]);
        if (lane == 0) red[w][k] = s;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int ww = 0; ww < kVT / 32; ww++) s += (double)red[ww][threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// cubic weight of tap k (0..3 = floor - 1 .. floor + 2) at fraction t, the same fp64
// expressions as cubic_w (so both adjoint forms use identical fp32 weights)
RS_DEV float cubic_tap(double t, int k) {
    const double A = -0.75;
    if (k == 1 || k == 2) {
        const double x = k == 1 ? t : 1.0 - t;
        return (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn(__dmul_rn(A + 2.0, x), A + 3.0), x), x), 1.0);
    }
    const double x = k == 0 ? t + 1.0 : 2.0 - t;
    return (float)__dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(A, x), 5.0 * A), x), 8.0 * A), x),
                            4.0 * A);
}

// red.global.add without a compiler memory clobber: the adjoint kernels below only read
// inputs that never alias the reduced output (API contract), so their loads may be
// scheduled across the reds
RS_DEV void red_add_nc(float *addr, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v));
}

// Real-arithmetic output -> input pixel map of sample n and its inverse (bounds only;
// membership is decided with the exact fp64 coordinate).
struct Aff {
    double m00, m01, m10, m11, p0x, p0y, i00, i01, i10, i11;
    bool ok;
};

RS_DEV Aff aff_of(const float *theta, int n, int H, int W, int Ho, int Wo, int ac) {
    const float *t = theta + 6 * n;
    const double t0 = __ldg(t), t1 = __ldg(t + 1), t2 = __ldg(t + 2), t3 = __ldg(t + 3), t4 = __ldg(t + 4),
                 t5 = __ldg(t + 5);
    const double ax = ac ? 2.0 / (Wo - 1) : 2.0 / Wo, bx = ac ? -1.0 : 1.0 / Wo - 1.0;
    const double ay = ac ? 2.0 / (Ho - 1) : 2.0 / Ho, by = ac ? -1.0 : 1.0 / Ho - 1.0;
    const double sx = ac ? 0.5 * (W - 1) : 0.5 * W, ox = ac ? 0.0 : -0.5;
    const double sy = ac ? 0.5 * (H - 1) : 0.5 * H, oy = ac ? 0.0 : -0.5;
    Aff A;
    A.m00 = sx * t0 * ax; A.m01 = sx * t1 * ay;
    A.m10 = sy * t3 * ax; A.m11 = sy * t4 * ay;
    A.p0x = sx * (t0 * bx + t1 * by + t2 + 1.0) + ox;
    A.p0y = sy * (t3 * bx + t4 * by + t5 + 1.0) + oy;
    const double det = A.m00 * A.m11 - A.m01 * A.m10;
    const double scale = fabs(A.m00 * A.m11) + fabs(A.m01 * A.m10);
    A.ok = isfinite(det) && fabs(det) > 1e-9 * (scale > 0 ? scale : 1.0) && fabs(det) > 1e-12;
    const double id = A.ok ? 1.0 / det : 0.0;
    A.i00 = A.m11 * id; A.i01 = -A.m01 * id;
    A.i10 = -A.m10 * id; A.i11 = A.m00 * id;
    return A;
}

constexpr int kGCH = 16;        // channels per pass of the bicubic gather
constexpr int kGWinMax = 1024;  // candidate output pixels per input pixel (else atomic)

// Bicubic d_input as a GATHER (scatter-to-gather by affine inversion):
// input pixel (x, y) collects the output pixels whose sample point lies in
// (x-2, x+2) x (y-2, y+2) -- the preimage of that square under the affine map,
// enumerated over its bounding box with exact fp64 membership.  Deterministic, no
// memset.  A sample whose map is singular or whose window is too large is flagged:
// its dX is zeroed here and bicubic_bwd adds it by reds.
// exact normalised coordinates of every output column / row (stn_norm has fp64 divisions)
__global__ void norm_tables(double *xt, double *yt, int Ho, int Wo, int ac) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Wo) xt[t] = stn_norm(t, Wo, ac);
    if (t < Ho) yt[t] = stn_norm(t, Ho, ac);
}

#ifndef RS_BC_GATHER_MINB
#define RS_BC_GATHER_MINB 2  // 128 registers (unbounded: 148, 1 block/SM; 930 vs 691 us)
#endif
__global__ void __launch_bounds__(kVT, RS_BC_GATHER_MINB)
    bicubic_dx_gather(StnArgs a, int *flags, const double *__restrict__ xtab, const double *__restrict__ ytab) {
    const int HW = a.H * a.W, P = a.Ho * a.Wo;
    const int n = blockIdx.y;
    const int idx = blockIdx.x * kVT + threadIdx.x;
    const Aff A = aff_of(a.theta, n, a.H, a.W, a.Ho, a.Wo, a.ac);
    const double eps = 1e-6;
    const double hj = 2.0 * (fabs(A.i00) + fabs(A.i01)) + eps, hi = 2.0 * (fabs(A.i10) + fabs(A.i11)) + eps;
    const bool ok = A.ok && (2.0 * hj + 2.0) * (2.0 * hi + 2.0) <= (double)kGWinMax;
    if (!ok && blockIdx.x == 0 && threadIdx.x == 0) flags[n] = 1;
    if (idx >= HW) return;
    const int y = idx / a.W, x = idx - y * a.W;
    float *dxn = a.dx + (long long)n * a.C * HW + idx;
    if (!ok) {
        for (int c = 0; c < a.C; c++) dxn[(long long)c * HW] = 0.f;
        return;
    }
    const float *t = a.theta + 6 * n;
    const double T0 = __ldg(t), T1 = __ldg(t + 1), T2 = __ldg(t + 2), T3 = __ldg(t + 3), T4 = __ldg(t + 4),
                 T5 = __ldg(t + 5);
    const double ux = (double)x - A.p0x, uy = (double)y - A.p0y;
    const double qj = A.i00 * ux + A.i01 * uy, qi = A.i10 * ux + A.i11 * uy;
    const int jlo = max(0, (int)ceil(qj - hj)), jhi = min(a.Wo - 1, (int)floor(qj + hj));
    const int ilo = max(0, (int)ceil(qi - hi)), ihi = min(a.Ho - 1, (int)floor(qi + hi));
    const float *gn = a.dy + (long long)n * a.C * P;
    for (int c0 = 0; c0 < a.C; c0 += kGCH) {
        float acc[kGCH];
#pragma unroll
        for (int c = 0; c < kGCH; c++) acc[c] = 0.f;
        for (int i = ilo; i <= ihi; i++) {
            const double yt = __ldg(ytab + i);
            for (int j = jlo; j <= jhi; j++) {
                const double xt = __ldg(xtab + j);
                const double ix = stn_unnorm(affine3(T0, T1, T2, xt, yt), a.W, a.ac);
                const double iy = stn_unnorm(affine3(T3, T4, T5, xt, yt), a.H, a.ac);
                const double fx = floor(ix), fy = floor(iy);
                const int kx = x - ((int)fx - 1), ky = y - ((int)fy - 1);
                if (kx < 0 || kx > 3 || ky < 0 || ky > 3) continue;
                const float w = cubic_tap(__dsub_rn(iy, fy), ky) * cubic_tap(__dsub_rn(ix, fx), kx);
                const float *g = gn + (long long)c0 * P + i * a.Wo + j;
#pragma unroll
                for (int c = 0; c < kGCH; c++)
                    if (c0 + c < a.C) acc[c] = fmaf(w, __ldg(g + (long long)c * P), acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < kGCH; c++)
            if (c0 + c < a.C) dxn[(long long)(c0 + c) * HW] = acc[c];
    }
}

#ifndef RS_BC_BWD_MINB
#define RS_BC_BWD_MINB 2  // 128 registers, no spills (3: 80 + 244 B spills, 662 vs 568 us)
#endif
__global__ void __launch_bounds__(kVT, RS_BC_BWD_MINB) bicubic_bwd(StnArgs a, double *part, const int *flags) {
    const int P = a.Ho * a.Wo, HW = a.H * a.W;
    const int q = out_pixel(a.Ho, a.Wo);
    const int n = blockIdx.y;
    if (flags && !flags[n]) a.dx = nullptr;  // d_input came from the gather
    float dth[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (q < P) {
        const int i = q / a.Wo, j = q - i * a.Wo;
        const Bicubic b = bicubic_at(a.theta, n, i, j, a.H, a.W, a.Ho, a.Wo, a.ac);
        // branch-free taps: out-of-image taps load from a clamped in-image address and the
        // value is then replaced by 0 (a select, so a non-finite neighbour cannot leak in),
        // so all 16 loads of a channel are issued together
        int ro[4], co[4];
        bool vy[4], vx[4];
        float wy[4], dwy[4], wx[4], dwx[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int yy = b.y0 - 1 + u, xx = b.x0 - 1 + u;
            vy[u] = yy >= 0 && yy < a.H;
            vx[u] = xx >= 0 && xx < a.W;
            ro[u] = (yy < 0 ? 0 : (yy >= a.H ? a.H - 1 : yy)) * a.W;
            co[u] = xx < 0 ? 0 : (xx >= a.W ? a.W - 1 : xx);
            wy[u] = vy[u] ? b.wy[u] : 0.f;
            dwy[u] = vy[u] ? b.dwy[u] : 0.f;
            wx[u] = vx[u] ? b.wx[u] : 0.f;
            dwx[u] = vx[u] ? b.dwx[u] : 0.f;
        }
        float gix = 0.f, giy = 0.f;
        for (int c = 0; c < a.C; c++) {
            const float g = __ldg(a.dy + ((long long)n * a.C + c) * P + q);
            const float *p = a.x + ((long long)n * a.C + c) * HW;
            if (a.dtheta) {
                float val[4][4];
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        const float t = __ldg(p + ro[u] + co[v]);
                        val[u][v] = (vy[u] && vx[v]) ? t : 0.f;
                    }
                float sx_ = 0.f, sy_ = 0.f;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    float rx = 0.f, ry = 0.f;
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        rx = fmaf(dwx[v], val[u][v], rx);
                        ry = fmaf(wx[v], val[u][v], ry);
                    }
                    sx_ = fmaf(wy[u], rx, sx_);
                    sy_ = fmaf(dwy[u], ry, sy_);
                }
                gix = fmaf(g, sx_, gix);
                giy = fmaf(g, sy_, giy);
            }
            if (a.dx) {
                float *d = a.dx + ((long long)n * a.C + c) * HW;
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int v = 0; v < 4; v++)
                        if (vy[u] && vx[v]) red_add_nc(d + ro[u] + co[v], g * (b.wy[u] * b.wx[v]));
            }
        }
        const float sx = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W, sy = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
        const float gx = gix * sx, gy = giy * sy, xt = (float)b.xt, yt = (float)b.yt;
        dth[0] = gx * xt; dth[1] = gx * yt; dth[2] = gx;
        dth[3] = gy * xt; dth[4] = gy * yt; dth[5] = gy;
    }
    if (a.dtheta) block_partial<6>(dth, part + ((long long)n * gridDim.x + blockIdx.x) * 6);
}

// ----------------------------------------------------------------- Lanczos-3
// 6 x 6 taps floor(i)-2 .. floor(i)+3, L(x) = sinc(x) sinc(x/3) (R13), weights
// and derivatives in fp64 (sinpi / cospi) rounded to fp32; same structure as the bicubic
// kernels with branch-free taps (clamped loads, out-of-image values selected to 0).
RS_DEV void lanczos_w(double t, float w[6], float dw[6]) {
    // x_m = t + 2 - m: sin(pi x_m) = (-1)^m sin(pi t) (likewise cos), and the x_m / 3 angles
    // step by -pi/3, so one sincospi pair per argument family serves all six taps
    const double pi = 3.14159265358979323846;
    const double cm[6] = {1.0, 0.5, -0.5, -1.0, -0.5, 0.5};  // cos(m pi / 3)
    const double sm[6] = {0.0, 0.86602540378443864676, 0.86602540378443864676, 0.0, -0.86602540378443864676,
                          -0.86602540378443864676};          // sin(m pi / 3)
    double s1, c1, sa, ca;
    sincospi(t, &s1, &c1);
    sincospi((t + 2.0) / 3.0, &sa, &ca);
#pragma unroll
    for (int m = 0; m < 6; m++) {
        const double x = t + 2.0 - m;
        if (x == 0.0) {
            w[m] = 1.f;
            dw[m] = 0.f;
        } else if (fabs(x) >= 3.0) {
            w[m] = 0.f;
            dw[m] = 0.f;
        } else {
            const double sg = (m & 1) ? -1.0 : 1.0;
            const double sx1 = sg * s1, cx1 = sg * c1;
            const double s3 = sa * cm[m] - ca * sm[m], c3 = ca * cm[m] + sa * sm[m];
            const double px = pi * x;
            w[m] = (float)(3.0 * sx1 * s3 / (px * px));
            dw[m] = (float)(3.0 * (pi * cx1 * s3 + (pi / 3.0) * sx1 * c3) / (px * px) - 6.0 * sx1 * s3 / (px * px * x));
        }
    }
}

struct Lz {
    int x0, y0;
    float wx[6], wy[6], dwx[6], dwy[6];
    double xt, yt;
};

RS_DEV Lz lanczos_at(const float *theta, int n, int i, int j, int H, int W, int Ho, int Wo, int ac) {
    Lz b;
    b.xt = stn_norm(j, Wo, ac);
    b.yt = stn_norm(i, Ho, ac);
    const float *t = theta + 6 * n;
    const double ix = stn_unnorm(affine3(__ldg(t), __ldg(t + 1), __ldg(t + 2), b.xt, b.yt), W, ac);
    const double iy = stn_unnorm(affine3(__ldg(t + 3), __ldg(t + 4), __ldg(t + 5), b.xt, b.yt), H, ac);
    const Cell cx = cell_of(ix), cy = cell_of(iy);
    b.x0 = cx.i0;
    b.y0 = cy.i0;
    lanczos_w(__dsub_rn(ix, floor(ix)), b.wx, b.dwx);
    lanczos_w(__dsub_rn(iy, floor(iy)), b.wy, b.dwy);
    return b;
}

#ifndef RS_LZ_MINB
#define RS_LZ_MINB 2
#endif
__global__ void __launch_bounds__(kVT, RS_LZ_MINB) lanczos_fwd(StnArgs a) {
    const int P = a.Ho * a.Wo, HW = a.H * a.W;
    const int q = out_pixel(a.Ho, a.Wo);
    if (q >= P) return;
    const int n = blockIdx.y, i = q / a.Wo, j = q - i * a.Wo;
    const Lz b = lanczos_at(a.theta, n, i, j, a.H, a.W, a.Ho, a.Wo, a.ac);
    int ro[6], co[6];
    bool vy[6], vx[6];
#pragma unroll
    for (int u = 0; u < 6; u++) {
        const int yy = b.y0 - 2 + u, xx = b.x0 - 2 + u;
        vy[u] = yy >= 0 && yy < a.H;
        vx[u] = xx >= 0 && xx < a.W;
        ro[u] = min(max(yy, 0), a.H - 1) * a.W;
        co[u] = min(max(xx, 0), a.W - 1);
    }
    for (int c = 0; c < a.C; c++) {
        const float *p = a.x + ((long long)n * a.C + c) * HW;
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < 6; u++) {
            float r = 0.f;
#pragma unroll
            for (int v = 0; v < 6; v++) {
                const float t = __ldg(p + ro[u] + co[v]);
                r = fmaf(b.wx[v], (vy[u] && vx[v]) ? t : 0.f, r);
            }
            s = fmaf(b.wy[u], r, s);
        }
        a.y[((long long)n * a.C + c) * P + q] = s;
    }
}

#ifndef RS_LZ_BWD_MINB
#define RS_LZ_BWD_MINB 1
#endif
__global__ void __launch_bounds__(kVT, RS_LZ_BWD_MINB) lanczos_bwd(StnArgs a, double *part) {
    const int P = a.Ho * a.Wo, HW = a.H * a.W;
    const int q = out_pixel(a.Ho, a.Wo);
    const int n = blockIdx.y;
    float dth[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (q < P) {
        const int i = q / a.Wo, j = q - i * a.Wo;
        const Lz b = lanczos_at(a.theta, n, i, j, a.H, a.W, a.Ho, a.Wo, a.ac);
        int ro[6], co[6];
        bool vy[6], vx[6];
#pragma unroll
        for (int u = 0; u < 6; u++) {
            const int yy = b.y0 - 2 + u, xx = b.x0 - 2 + u;
            vy[u] = yy >= 0 && yy < a.H;
            vx[u] = xx >= 0 && xx < a.W;
            ro[u] = min(max(yy, 0), a.H - 1) * a.W;
            co[u] = min(max(xx, 0), a.W - 1);
        }
        float gix = 0.f, giy = 0.f;
        for (int c = 0; c < a.C; c++) {
            const float g = __ldg(a.dy + ((long long)n * a.C + c) * P + q);
            const float *p = a.x + ((long long)n * a.C + c) * HW;
            if (a.dtheta) {
                float sx_ = 0.f, sy_ = 0.f;
#pragma unroll
                for (int u = 0; u < 6; u++) {
                    float rx = 0.f, ry = 0.f;
#pragma unroll
                    for (int v = 0; v < 6; v++) {
                        const float t = __ldg(p + ro[u] + co[v]);
                        const float val = (vy[u] && vx[v]) ? t : 0.f;
                        rx = fmaf(b.dwx[v], val, rx);
                        ry = fmaf(b.wx[v], val, ry);
                    }
                    sx_ = fmaf(b.wy[u], rx, sx_);
                    sy_ = fmaf(b.dwy[u], ry, sy_);
                }
                gix = fmaf(g, sx_, gix);
                giy = fmaf(g, sy_, giy);
            }
            if (a.dx) {
                float *d = a.dx + ((long long)n * a.C + c) * HW;
#pragma unroll
                for (int u = 0; u < 6; u++) {
                    const float gw = g * b.wy[u];
#pragma unroll
                    for (int v = 0; v < 6; v++)
                        if (vy[u] && vx[v]) red_add_nc(d + ro[u] + co[v], gw * b.wx[v]);
                }
            }
        }
        const float sx = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W, sy = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
        const float gx = gix * sx, gy = giy * sy, xt = (float)b.xt, yt = (float)b.yt;
        dth[0] = gx * xt; dth[1] = gx * yt; dth[2] = gx;
        dth[3] = gy * xt; dth[4] = gy * yt; dth[5] = gy;
    }
    if (a.dtheta) block_partial<6>(dth, part + ((long long)n * gridDim.x + blockIdx.x) * 6);
}

// ----------------------------------------------------------------- 3-D
struct Vol {
    int N, C, D, H, W, Do, Ho, Wo, ac;
    const float *x, *theta, *dy;
    float *y, *dx, *dtheta;
};

struct Tri {
    int x0, y0, z0;
    float f[3];
    double t[3];
};

RS_DEV Tri tri_at(const Vol &a, int n, int k, int i, int j) {
    Tri r;
    r.t[0] = stn_norm(j, a.Wo, a.ac);
    r.t[1] = stn_norm(i, a.Ho, a.ac);
    r.t[2] = stn_norm(k, a.Do, a.ac);
    const float *th = a.theta + 12 * n;
    const int L[3] = {a.W, a.H, a.D};
    int c0[3];
#pragma unroll
    for (int d = 0; d < 3; d++) {
        // ((t0 x + t1 y) + t2 z) + t3, the oracle's order
        const double g = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__ldg(th + 4 * d), r.t[0]),
                                                       __dmul_rn(__ldg(th + 4 * d + 1), r.t[1])),
                                             __dmul_rn(__ldg(th + 4 * d + 2), r.t[2])),
                                   (double)__ldg(th + 4 * d + 3));
        const double pcoord = stn_unnorm(g, L[d], a.ac);
        const Cell cc = cell_of(pcoord);
        c0[d] = cc.i0;
        r.f[d] = cc.f;
    }
    r.x0 = c0[0];
    r.y0 = c0[1];
    r.z0 = c0[2];
    return r;
}

__global__ void __launch_bounds__(kVT) stn3d_fwd_k(Vol a) {
    const int P = a.Do * a.Ho * a.Wo;
    const long long V = (long long)a.D * a.H * a.W;
    const int q = blockIdx.x * kVT + threadIdx.x;
    if (q >= P) return;
    const int n = blockIdx.y;
    const int k = q / (a.Ho * a.Wo), rem = q - k * a.Ho * a.Wo, i = rem / a.Wo, j = rem - i * a.Wo;
    const Tri r = tri_at(a, n, k, i, j);
    for (int c = 0; c < a.C; c++) {
        const float *p = a.x + ((long long)n * a.C + c) * V;
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const int ax = e & 1, by = (e >> 1) & 1, dz = e >> 2;
            const int xx = r.x0 + ax, yy = r.y0 + by, zz = r.z0 + dz;
            if (xx < 0 || xx >= a.W || yy < 0 || yy >= a.H || zz < 0 || zz >= a.D) continue;
            const float w = (ax ? r.f[0] : 1.f - r.f[0]) * (by ? r.f[1] : 1.f - r.f[1]) * (dz ? r.f[2] : 1.f - r.f[2]);
            s = fmaf(w, __ldg(p + ((long long)zz * a.H + yy) * a.W + xx), s);
        }
        a.y[((long long)n * a.C + c) * P + q] = s;
    }
}

__global__ void __launch_bounds__(kVT, 3) stn3d_bwd_k(Vol a, double *part) {
    const int P = a.Do * a.Ho * a.Wo;
    const long long V = (long long)a.D * a.H * a.W;
    const int q = blockIdx.x * kVT + threadIdx.x;
    const int n = blockIdx.y;
    float dth[12];
#pragma unroll
    for (int e = 0; e < 12; e++) dth[e] = 0.f;
    if (q < P) {
        const int k = q / (a.Ho * a.Wo), rem = q - k * a.Ho * a.Wo, i = rem / a.Wo, j = rem - i * a.Wo;
        const Tri r = tri_at(a, n, k, i, j);
        // branch-free taps (as bicubic_bwd): clamped loads, out-of-volume values selected to 0
        long long off[8];
        bool ok[8];
        float w[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const int ax = e & 1, by = (e >> 1) & 1, dz = e >> 2;
            const int xx = r.x0 + ax, yy = r.y0 + by, zz = r.z0 + dz;
            ok[e] = xx >= 0 && xx < a.W && yy >= 0 && yy < a.H && zz >= 0 && zz < a.D;
            const int xc = min(max(xx, 0), a.W - 1), yc = min(max(yy, 0), a.H - 1), zc = min(max(zz, 0), a.D - 1);
            off[e] = ((long long)zc * a.H + yc) * a.W + xc;
            w[e] = (ax ? r.f[0] : 1.f - r.f[0]) * (by ? r.f[1] : 1.f - r.f[1]) * (dz ? r.f[2] : 1.f - r.f[2]);
        }
        float gq[3] = {0.f, 0.f, 0.f};
        for (int c = 0; c < a.C; c++) {
            const float g = __ldg(a.dy + ((long long)n * a.C + c) * P + q);
            const float *p = a.x + ((long long)n * a.C + c) * V;
            if (a.dtheta) {
                float v[8];
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const float t = __ldg(p + off[e]);
                    v[e] = ok[e] ? t : 0.f;
                }
                const float wx0 = 1.f - r.f[0], wx1 = r.f[0], wy0 = 1.f - r.f[1], wy1 = r.f[1];
                const float wz0 = 1.f - r.f[2], wz1 = r.f[2];
                // e = ax + 2 by + 4 dz: d/dx pairs (e, e+1), d/dy (e, e+2), d/dz (e, e+4)
                const float gx_ = wz0 * (wy0 * (v[1] - v[0]) + wy1 * (v[3] - v[2])) +
                                  wz1 * (wy0 * (v[5] - v[4]) + wy1 * (v[7] - v[6]));
                const float gy_ = wz0 * (wx0 * (v[2] - v[0]) + wx1 * (v[3] - v[1])) +
                                  wz1 * (wx0 * (v[6] - v[4]) + wx1 * (v[7] - v[5]));
                const float gz_ = wy0 * (wx0 * (v[4] - v[0]) + wx1 * (v[5] - v[1])) +
                                  wy1 * (wx0 * (v[6] - v[2]) + wx1 * (v[7] - v[3]));
                gq[0] = fmaf(g, gx_, gq[0]);
                gq[1] = fmaf(g, gy_, gq[1]);
                gq[2] = fmaf(g, gz_, gq[2]);
            }
            if (a.dx) {
                float *d = a.dx + ((long long)n * a.C + c) * V;
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if (ok[e]) red_add_nc(d + off[e], g * w[e]);
            }
        }
        const int L[3] = {a.W, a.H, a.D};
#pragma unroll
        for (int d = 0; d < 3; d++) {
            const float gg = gq[d] * (a.ac ? 0.5f * (L[d] - 1) : 0.5f * L[d]);
            dth[4 * d] = gg * (float)r.t[0];
            dth[4 * d + 1] = gg * (float)r.t[1];
            dth[4 * d + 2] = gg * (float)r.t[2];
            dth[4 * d + 3] = gg;
        }
    }
    if (a.dtheta) block_partial<12>(dth, part + ((long long)n * gridDim.x + blockIdx.x) * 12);
}

// dtheta[n][e] = fixed-order fp64 sum over the sample's block partials
__global__ void theta_finalize(const double *part, int nb, int ne, float *dtheta) {
    const int n = blockIdx.x, e = threadIdx.x;
    if (e >= ne) return;
    double s = 0.0;
    for (int b = 0; b < nb; b++) s += part[((long long)n * nb + b) * ne + e];
    dtheta[n * ne + e] = (float)s;
}

// Bicubic taps for the deterministic fixed-point scatter (det.cuh): the 16 in-image
// taps of bicubic_bwd with its fp32 weights wy * wx (|w| <= 1 per tap).
struct BicubicTapSampler {
    const float *theta;
    int H, W, Ho, Wo, ac;
    static constexpr int kMaxTaps = 16;
    static constexpr double kWmax = 1.0;
    RS_DEV int taps(int n, long long q, long long *off, float *w) const {
        const int i = (int)(q / Wo), j = (int)(q - (long long)i * Wo);
        const Bicubic b = bicubic_at(theta, n, i, j, H, W, Ho, Wo, ac);
        int k = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int yy = b.y0 - 1 + u;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const int xx = b.x0 - 1 + v;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
                    off[k] = (long long)yy * W + xx;
                    w[k++] = b.wy[u] * b.wx[v];
                }
            }
        }
        return k;
    }
};

// Lanczos-3 taps for the fixed-point scatter: the 36 in-image taps of lanczos_bwd with its
// fp32 weights wy * wx (|L| <= 1, so |w| <= 1 per tap and per element sum_q |w| <= P).
struct LanczosTapSampler {
    const float *theta;
    int H, W, Ho, Wo, ac;
    static constexpr int kMaxTaps = 36;
    static constexpr double kWmax = 1.0;
    RS_DEV int taps(int n, long long q, long long *off, float *w) const {
        const int i = (int)(q / Wo), j = (int)(q - (long long)i * Wo);
        const Lz b = lanczos_at(theta, n, i, j, H, W, Ho, Wo, ac);
        int k = 0;
#pragma unroll
        for (int u = 0; u < 6; u++) {
            const int yy = b.y0 - 2 + u;
#pragma unroll
            for (int v = 0; v < 6; v++) {
                const int xx = b.x0 - 2 + v;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
                    off[k] = (long long)yy * W + xx;
                    w[k++] = b.wy[u] * b.wx[v];
                }
            }
        }
        return k;
    }
};

// Trilinear 3-D taps for the fixed-point scatter: the 8 in-volume taps of stn3d_bwd_k.
struct Vol3dTapSampler {
    Vol a;
    static constexpr int kMaxTaps = 8;
    static constexpr double kWmax = 1.0;
    RS_DEV int taps(int n, long long q, long long *off, float *w) const {
        const int k0 = (int)(q / ((long long)a.Ho * a.Wo));
        const int rem = (int)(q - (long long)k0 * a.Ho * a.Wo), i = rem / a.Wo, j = rem - i * a.Wo;
        const Tri r = tri_at(a, n, k0, i, j);
        int k = 0;
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const int ax = e & 1, by = (e >> 1) & 1, dz = e >> 2;
            const int xx = r.x0 + ax, yy = r.y0 + by, zz = r.z0 + dz;
            if (xx >= 0 && xx < a.W && yy >= 0 && yy < a.H && zz >= 0 && zz < a.D) {
                off[k] = ((long long)zz * a.H + yy) * a.W + xx;
                w[k++] = (ax ? r.f[0] : 1.f - r.f[0]) * (by ? r.f[1] : 1.f - r.f[1]) * (dz ? r.f[2] : 1.f - r.f[2]);
            }
        }
        return k;
    }
};

}  // namespace

size_t stn_var_ws_bytes(int N, int P, int ne) {
    return sizeof(double) * (size_t)N * ((P + kVT - 1) / kVT) * ne;
}

static size_t bicubic_base_bytes(int N, int Ho, int Wo) {
    return det_align(stn_var_ws_bytes(N, Ho * Wo, 6) + sizeof(double) * (size_t)(Ho + Wo) + sizeof(int) * (size_t)N);
}

size_t stn_bicubic_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det) {
    return bicubic_base_bytes(N, Ho, Wo) + (det ? det_ws_bytes(N, (long long)C * H * W) : 0);
}

cudaError_t stn_bicubic_launch(const StnArgs &a, bool bwd, int algo, bool det, void *ws, cudaStream_t s) {
    const int P = a.Ho * a.Wo;
    const dim3 grid((P + kVT - 1) / kVT, a.N);
    if (!bwd) {
        bicubic_fwd<<<grid, kVT, 0, s>>>(a);
        note_launch();
        return cudaGetLastError();
    }
    // workspace: d_theta partials, then one flag per sample (gather fallback)
    // workspace: d_theta partials | xt[Wo], yt[Ho] | one flag per sample
    double *part = (double *)ws;
    double *xtab = part + stn_var_ws_bytes(a.N, P, 6) / sizeof(double), *ytab = xtab + a.Wo;
    int *flags = (int *)(ytab + a.Ho);
    // GATHER (or deterministic=1, passed as algo 1): the converted gather; AUTO takes the
    // atomic scatter, measured faster here (4 x 16 x 512^2: 0.79 ms for reds + d_theta in
    // one pass vs 0.57 ms gather + 0.28 ms d_theta pass)
    const bool gather = a.dx && (algo == 1 /*GATHER*/ || det);
    if (gather) {
        cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)a.N, s);
        if (e != cudaSuccess) return e;
        const int nt = a.Ho > a.Wo ? a.Ho : a.Wo;
        norm_tables<<<(nt + 255) / 256, 256, 0, s>>>(xtab, ytab, a.Ho, a.Wo, a.ac);
        note_launch();
        const int HW = a.H * a.W;
        bicubic_dx_gather<<<dim3((HW + kVT - 1) / kVT, a.N), kVT, 0, s>>>(a, flags, xtab, ytab);
        note_launch();
    } else if (a.dx) {
        cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * a.H * a.W, s);
        if (e != cudaSuccess) return e;
    }
    if (det && gather) {
        // deterministic=1: d_theta for every sample here, the gather's fallback samples'
        // d_input (flags[n] = 1) by the fixed-point scatter instead of reds
        StnArgs b = a;
        b.dx = nullptr;
        if (a.dtheta) {
            bicubic_bwd<<<grid, kVT, 0, s>>>(b, part, nullptr);
            note_launch();
        }
        const BicubicTapSampler smp{a.theta, a.H, a.W, a.Ho, a.Wo, a.ac};
        cudaError_t e = det_scatter_launch(smp, a.dy, a.dx, a.N, a.C, (long long)a.H * a.W, (long long)P, nullptr,
                                           nullptr, flags, (char *)ws + bicubic_base_bytes(a.N, a.Ho, a.Wo), s);
        if (e != cudaSuccess) return e;
    } else {
        bicubic_bwd<<<grid, kVT, 0, s>>>(a, part, gather ? flags : nullptr);
        note_launch();
    }
    if (a.dtheta) {
        theta_finalize<<<a.N, 32, 0, s>>>(part, grid.x, 6, a.dtheta);
        note_launch();
    }
    return cudaGetLastError();
}

size_t stn_lanczos_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det) {
    return det_align(stn_var_ws_bytes(N, Ho * Wo, 6)) + (det ? det_ws_bytes(N, (long long)C * H * W) : 0);
}

size_t stn3d_ws_bytes(int N, int C, int D, int H, int W, int Do, int Ho, int Wo, bool det) {
    return det_align(stn_var_ws_bytes(N, Do * Ho * Wo, 12)) + (det ? det_ws_bytes(N, (long long)C * D * H * W) : 0);
}

cudaError_t stn_lanczos_launch(const StnArgs &a, bool bwd, bool det, void *ws, cudaStream_t s) {
    const int P = a.Ho * a.Wo;
    const dim3 grid((P + kVT - 1) / kVT, a.N);
    if (!bwd) {
        lanczos_fwd<<<grid, kVT, 0, s>>>(a);
        note_launch();
        return cudaGetLastError();
    }
    if (det && a.dx) {  // deterministic=1: d_theta pass alone, then the fixed-point scatter
        if (a.dtheta) {
            StnArgs b = a;
            b.dx = nullptr;
            cudaError_t e = stn_lanczos_launch(b, true, false, ws, s);
            if (e != cudaSuccess) return e;
        }
        const LanczosTapSampler smp{a.theta, a.H, a.W, a.Ho, a.Wo, a.ac};
        return det_scatter_launch(smp, a.dy, a.dx, a.N, a.C, (long long)a.H * a.W, (long long)P, nullptr, nullptr,
                                  nullptr, (char *)ws + det_align(stn_var_ws_bytes(a.N, P, 6)), s);
    }
    if (a.dx) {
        cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * a.H * a.W, s);
        if (e != cudaSuccess) return e;
    }
    lanczos_bwd<<<grid, kVT, 0, s>>>(a, (double *)ws);
    note_launch();
    if (a.dtheta) {
        theta_finalize<<<a.N, 32, 0, s>>>((const double *)ws, grid.x, 6, a.dtheta);
        note_launch();
    }
    return cudaGetLastError();
}

cudaError_t stn3d_launch(const float *x, const float *theta, const float *dy, float *y, float *dx, float *dtheta,
                         int N, int C, int D, int H, int W, int Do, int Ho, int Wo, int ac, bool bwd, bool det,
                         void *ws, cudaStream_t s) {
    Vol a{N, C, D, H, W, Do, Ho, Wo, ac, x, theta, dy, y, dx, dtheta};
    const int P = Do * Ho * Wo;
    const dim3 grid((P + kVT - 1) / kVT, N);
    if (!bwd) {
        stn3d_fwd_k<<<grid, kVT, 0, s>>>(a);
        note_launch();
        return cudaGetLastError();
    }
    if (det && dx) {  // deterministic=1: d_theta pass alone, then the fixed-point scatter
        if (dtheta) {
            cudaError_t e = stn3d_launch(x, theta, dy, y, nullptr, dtheta, N, C, D, H, W, Do, Ho, Wo, ac, true, false,
                                         ws, s);
            if (e != cudaSuccess) return e;
        }
        const Vol3dTapSampler smp{a};
        return det_scatter_launch(smp, dy, dx, N, C, (long long)D * H * W, (long long)P, nullptr, nullptr, nullptr,
                                  (char *)ws + det_align(stn_var_ws_bytes(N, P, 12)), s);
    }
    if (dx) {
        cudaError_t e = cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)N * C * D * H * W, s);
        if (e != cudaSuccess) return e;
    }
    stn3d_bwd_k<<<grid, kVT, 0, s>>>(a, (double *)ws);
    note_launch();
    if (dtheta) {
        theta_finalize<<<N, 32, 0, s>>>((const double *)ws, grid.x, 12, dtheta);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace rs
