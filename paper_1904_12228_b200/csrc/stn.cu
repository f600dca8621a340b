// stn.cu — spatial transformer (affine_grid + bilinear grid_sample), forward and
// adjoint, sm_100a.  PAPER.md:21-28 (layer), PAPER.md:700-733 (scatter-to-gather
// conversion vs atomics), PAPER.md:838-840 (reductions: partial + serial).
//
// Kernels
//   stn_fwd_kernel          one thread per output pixel, all channels; the
//                           sampling grid is never materialised (K1).
//   stn_tables_kernel       xt[Wo], yt[Ho] in fp64 (exact, shared by the bwd).
//   stn_dtheta_kernel       per output pixel d_ix/d_iy over channels, then the
//                           6 theta terms reduced warp -> block (fp32) -> fp64
//                           per-block partials (rfactor-style).
//   stn_dtheta_finalize     per-sample fixed-order fp64 sum of the partials.
//   stn_dx_gather_kernel    scatter-to-gather by affine inversion: each input
//                           pixel walks the bounding box of its preimage in
//                           output space and re-derives which outputs sample
//                           it; deterministic, no memset.
//   stn_dx_scatter_kernel   atomic scatter fallback: border
//                           padding, near-singular theta, or forced.
#include "common.cuh"

namespace rs {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGatherCand = 256;  // preimage bbox budget per input pixel

struct Theta {
    double t[6];
};

RS_DEV Theta load_theta(const float *theta, int n) {
    Theta T;
#pragma unroll
    for (int k = 0; k < 6; k++) T.t[k] = (double)__ldg(theta + 6 * n + k);
    return T;
}

// Sample coordinate of output (i, j) given its normalised coords.
RS_DEV void stn_coord(const Theta &T, double xt, double yt, int H, int W, int ac, double &ix,
                      double &iy) {
    ix = stn_unnorm(affine3(T.t[0], T.t[1], T.t[2], xt, yt), W, ac);
    iy = stn_unnorm(affine3(T.t[3], T.t[4], T.t[5], xt, yt), H, ac);
}

// Affine map q=(j,i) -> p=(ix,iy) in real arithmetic (for the preimage bbox
// only; membership is always re-decided with the exact fp64 coordinate).
struct AffineInv {
    double m00, m01, m10, m11;  // inverse of d p / d q
    double p0x, p0y;            // p at q = 0
    double hj, hi;              // half extents of the preimage of a 2x2 px square
    bool ok;
};

RS_DEV AffineInv stn_inverse(const Theta &T, int H, int W, int Ho, int Wo, int ac) {
    double ax = ac ? 2.0 / (Wo - 1) : 2.0 / Wo, bx = ac ? -1.0 : 1.0 / Wo - 1.0;
    double ay = ac ? 2.0 / (Ho - 1) : 2.0 / Ho, by = ac ? -1.0 : 1.0 / Ho - 1.0;
    double sx = ac ? 0.5 * (W - 1) : 0.5 * W, ox = ac ? 0.0 : -0.5;
    double sy = ac ? 0.5 * (H - 1) : 0.5 * H, oy = ac ? 0.0 : -0.5;
    double a00 = sx * T.t[0] * ax, a01 = sx * T.t[1] * ay;
    double a10 = sy * T.t[3] * ax, a11 = sy * T.t[4] * ay;
    AffineInv r;
    r.p0x = sx * (T.t[0] * bx + T.t[1] * by + T.t[2] + 1.0) + ox;
    r.p0y = sy * (T.t[3] * bx + T.t[4] * by + T.t[5] + 1.0) + oy;
    double det = a00 * a11 - a01 * a10;
    double scale = fabs(a00 * a11) + fabs(a01 * a10);
    r.ok = isfinite(det) && fabs(det) > 1e-9 * (scale > 0 ? scale : 1.0) && fabs(det) > 1e-12;
    if (!r.ok) {
        r.m00 = r.m01 = r.m10 = r.m11 = r.hj = r.hi = 0.0;
        return r;
    }
    double id = 1.0 / det;
    r.m00 = a11 * id;
    r.m01 = -a01 * id;
    r.m10 = -a10 * id;
    r.m11 = a00 * id;
    r.hj = fabs(r.m00) + fabs(r.m01);
    r.hi = fabs(r.m10) + fabs(r.m11);
    double cand = (2.0 * r.hj + 2.0) * (2.0 * r.hi + 2.0);
    if (!(cand <= (double)kMaxGatherCand)) r.ok = false;
    return r;
}

// ----------------------------------------------------------------- forward
__global__ void __launch_bounds__(kThreads) stn_fwd_kernel(StnArgs a) {
    const long long P = (long long)a.Ho * a.Wo;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= (long long)a.N * P) return;
    const int n = (int)(idx / P);
    const long long rem = idx - (long long)n * P;
    const int i = (int)(rem / a.Wo), j = (int)(rem - (long long)i * a.Wo);
    const Theta T = load_theta(a.theta, n);
    double ix, iy;
    stn_coord(T, stn_norm(j, a.Wo, a.ac), stn_norm(i, a.Ho, a.ac), a.H, a.W, a.ac, ix, iy);
    if (a.border) {
        float d;
        ix = clamp_coord(ix, a.W, d);
        iy = clamp_coord(iy, a.H, d);
    }
    const Cell cx = cell_of(ix), cy = cell_of(iy);
    const bool x0ok = cx.i0 >= 0 && cx.i0 < a.W, x1ok = cx.i0 + 1 >= 0 && cx.i0 + 1 < a.W;
    const bool y0ok = cy.i0 >= 0 && cy.i0 < a.H, y1ok = cy.i0 + 1 >= 0 && cy.i0 + 1 < a.H;
    const float wx0 = 1.f - cx.f, wx1 = cx.f, wy0 = 1.f - cy.f, wy1 = cy.f;
    const float w00 = wy0 * wx0, w01 = wy0 * wx1, w10 = wy1 * wx0, w11 = wy1 * wx1;
    const long long HW = (long long)a.H * a.W;
    const long long o00 = (long long)cy.i0 * a.W + cx.i0;
    const bool k00 = y0ok && x0ok, k01 = y0ok && x1ok, k10 = y1ok && x0ok, k11 = y1ok && x1ok;
    const float *xp = a.x + (long long)n * a.C * HW;
    float *yp = a.y + (long long)n * a.C * P + rem;
#pragma unroll 4
    for (int c = 0; c < a.C; c++) {
        const float *p = xp + (long long)c * HW + o00;
        float v = 0.f;
        if (k00) v = fmaf(w00, __ldg(p), v);
        if (k01) v = fmaf(w01, __ldg(p + 1), v);
        if (k10) v = fmaf(w10, __ldg(p + a.W), v);
        if (k11) v = fmaf(w11, __ldg(p + a.W + 1), v);
        yp[(long long)c * P] = v;
    }
}

// ----------------------------------------------------------------- backward: tables
__global__ void stn_tables_kernel(double *xt, double *yt, int Ho, int Wo, int ac) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Wo) xt[t] = stn_norm(t, Wo, ac);
    if (t < Ho) yt[t] = stn_norm(t, Ho, ac);
}

// ----------------------------------------------------------------- backward: d_theta
__global__ void __launch_bounds__(kThreads)
    stn_dtheta_kernel(StnArgs a, const double *__restrict__ xtab, const double *__restrict__ ytab,
                      double *__restrict__ partials, int bps) {
    const int n = blockIdx.y;
    const long long P = (long long)a.Ho * a.Wo;
    const long long HW = (long long)a.H * a.W;
    const Theta T = load_theta(a.theta, n);
    const float sx = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W;
    const float sy = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
    const float *xp = a.x + (long long)n * a.C * HW;
    const float *gp = a.dy + (long long)n * a.C * P;
    float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (long long p = (long long)blockIdx.x * kThreads + threadIdx.x; p < P;
         p += (long long)bps * kThreads) {
        const int i = (int)(p / a.Wo), j = (int)(p - (long long)i * a.Wo);
        const double xt = xtab[j], yt = ytab[i];
        double ix, iy;
        stn_coord(T, xt, yt, a.H, a.W, a.ac, ix, iy);
        float cgx = 1.f, cgy = 1.f;
        if (a.border) {
            ix = clamp_coord(ix, a.W, cgx);
            iy = clamp_coord(iy, a.H, cgy);
        }
        const Cell cx = cell_of(ix), cy = cell_of(iy);
        const bool x0ok = cx.i0 >= 0 && cx.i0 < a.W, x1ok = cx.i0 + 1 >= 0 && cx.i0 + 1 < a.W;
        const bool y0ok = cy.i0 >= 0 && cy.i0 < a.H, y1ok = cy.i0 + 1 >= 0 && cy.i0 + 1 < a.H;
        const bool k00 = y0ok && x0ok, k01 = y0ok && x1ok, k10 = y1ok && x0ok, k11 = y1ok && x1ok;
        const long long o00 = (long long)cy.i0 * a.W + cx.i0;
        const float fx = cx.f, fy = cy.f;
        float dix = 0.f, diy = 0.f;
#pragma unroll 4
        for (int c = 0; c < a.C; c++) {
            const float *q = xp + (long long)c * HW + o00;
            const float g = ldg_stream(gp + (long long)c * P + p);
            const float v00 = k00 ? __ldg(q) : 0.f, v01 = k01 ? __ldg(q + 1) : 0.f;
            const float v10 = k10 ? __ldg(q + a.W) : 0.f, v11 = k11 ? __ldg(q + a.W + 1) : 0.f;
            dix = fmaf(g, fmaf(1.f - fy, v01 - v00, fy * (v11 - v10)), dix);
            diy = fmaf(g, fmaf(1.f - fx, v10 - v00, fx * (v11 - v01)), diy);
        }
        const float dgx = dix * sx * cgx, dgy = diy * sy * cgy;
        const float fxt = (float)xt, fyt = (float)yt;
        acc[0] = fmaf(dgx, fxt, acc[0]);
        acc[1] = fmaf(dgx, fyt, acc[1]);
        acc[2] += dgx;
        acc[3] = fmaf(dgy, fxt, acc[3]);
        acc[4] = fmaf(dgy, fyt, acc[4]);
        acc[5] += dgy;
    }
    __shared__ float red[kThreads / 32][6];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; k++) {
        float v = warp_sum(acc[k]);
        if (lane == 0) red[wid][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; w++) s += (double)red[w][threadIdx.x];
        partials[((long long)n * bps + blockIdx.x) * 6 + threadIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kThreads)
    stn_dtheta_finalize(const double *__restrict__ partials, int bps, float *dtheta) {
    const int n = blockIdx.x;
    __shared__ double red[kThreads / 32][6];
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < bps; b += kThreads)
#pragma unroll
        for (int k = 0; k < 6; k++) s[k] += partials[((long long)n * bps + b) * 6 + k];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; k++) {
        double v = warp_sum_d(s[k]);
        if (lane == 0) red[wid][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = 0.0;
        for (int w = 0; w < kThreads / 32; w++) v += red[w][threadIdx.x];
        dtheta[6 * n + threadIdx.x] = (float)v;
    }
}

// ----------------------------------------------------------------- backward: dx, gather form
// CT channels per pass over the preimage bbox.
template <int CT>
__global__ void __launch_bounds__(kThreads)
    stn_dx_gather_kernel(StnArgs a, const double *__restrict__ xtab,
                         const double *__restrict__ ytab) {
    const long long HW = (long long)a.H * a.W;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= (long long)a.N * HW) return;
    const int n = (int)(idx / HW);
    const long long rem = idx - (long long)n * HW;
    const int y = (int)(rem / a.W), x = (int)(rem - (long long)y * a.W);
    const Theta T = load_theta(a.theta, n);
    const AffineInv inv = stn_inverse(T, a.H, a.W, a.Ho, a.Wo, a.ac);
    float *dxp = a.dx + (long long)n * a.C * HW + rem;
    if (!inv.ok) {  // this sample takes the atomic scatter: zero-fill for it
        for (int c = 0; c < a.C; c++) dxp[(long long)c * HW] = 0.f;
        return;
    }
    // preimage of p in [x-1, x+1] x [y-1, y+1]
    const double ux = (double)x - inv.p0x, uy = (double)y - inv.p0y;
    const double qj = inv.m00 * ux + inv.m01 * uy, qi = inv.m10 * ux + inv.m11 * uy;
    const double mj = inv.hj + 1e-3, mi = inv.hi + 1e-3;
    const int jlo = max(0, (int)ceil(qj - mj)), jhi = min(a.Wo - 1, (int)floor(qj + mj));
    const int ilo = max(0, (int)ceil(qi - mi)), ihi = min(a.Ho - 1, (int)floor(qi + mi));
    const long long P = (long long)a.Ho * a.Wo;
    const float *gp = a.dy + (long long)n * a.C * P;
    for (int cb = 0; cb < a.C; cb += CT) {
        float acc[CT];
#pragma unroll
        for (int c = 0; c < CT; c++) acc[c] = 0.f;
        for (int i = ilo; i <= ihi; i++) {
            const double yt = ytab[i];
            const double t1y = __dmul_rn(T.t[1], yt), t4y = __dmul_rn(T.t[4], yt);
            for (int j = jlo; j <= jhi; j++) {
                const double xt = xtab[j];
                const double ix = stn_unnorm(
                    __dadd_rn(__dadd_rn(__dmul_rn(T.t[0], xt), t1y), T.t[2]), a.W, a.ac);
                const double iy = stn_unnorm(
                    __dadd_rn(__dadd_rn(__dmul_rn(T.t[3], xt), t4y), T.t[5]), a.H, a.ac);
                const Cell cx = cell_of(ix), cy = cell_of(iy);
                const bool hx = (cx.i0 == x) || (cx.i0 == x - 1);
                const bool hy = (cy.i0 == y) || (cy.i0 == y - 1);
                if (!(hx && hy)) continue;
                const float wx = (cx.i0 == x) ? 1.f - cx.f : cx.f;
                const float wy = (cy.i0 == y) ? 1.f - cy.f : cy.f;
                const float w = wy * wx;
                const float *g = gp + (long long)i * a.Wo + j + (long long)cb * P;
#pragma unroll
                for (int c = 0; c < CT; c++)
                    if (cb + c < a.C) acc[c] = fmaf(w, __ldg(g + (long long)c * P), acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < CT; c++)
            if (cb + c < a.C) dxp[(long long)(cb + c) * HW] = acc[c];
    }
}

// ----------------------------------------------------------------- backward: dx, atomic scatter
// only_nongather: skip samples the gather kernel handled (AUTO).  Grid is
// (blocks per sample, N) so a skipped sample costs one early-exit per block.
__global__ void __launch_bounds__(kThreads) stn_dx_scatter_kernel(StnArgs a, int only_nongather) {
    const int n = blockIdx.y;
    const Theta T = load_theta(a.theta, n);
    if (only_nongather && stn_inverse(T, a.H, a.W, a.Ho, a.Wo, a.ac).ok) return;
    const long long P = (long long)a.Ho * a.Wo;
    const long long HW = (long long)a.H * a.W;
    for (long long rem = (long long)blockIdx.x * kThreads + threadIdx.x; rem < P;
         rem += (long long)gridDim.x * kThreads) {
        const int i = (int)(rem / a.Wo), j = (int)(rem - (long long)i * a.Wo);
        double ix, iy;
        stn_coord(T, stn_norm(j, a.Wo, a.ac), stn_norm(i, a.Ho, a.ac), a.H, a.W, a.ac, ix, iy);
        if (a.border) {
            float d;
            ix = clamp_coord(ix, a.W, d);
            iy = clamp_coord(iy, a.H, d);
        }
        const Cell cx = cell_of(ix), cy = cell_of(iy);
        const bool x0ok = cx.i0 >= 0 && cx.i0 < a.W, x1ok = cx.i0 + 1 >= 0 && cx.i0 + 1 < a.W;
        const bool y0ok = cy.i0 >= 0 && cy.i0 < a.H, y1ok = cy.i0 + 1 >= 0 && cy.i0 + 1 < a.H;
        const float wx0 = 1.f - cx.f, wx1 = cx.f, wy0 = 1.f - cy.f, wy1 = cy.f;
        const float w00 = wy0 * wx0, w01 = wy0 * wx1, w10 = wy1 * wx0, w11 = wy1 * wx1;
        const long long o00 = (long long)cy.i0 * a.W + cx.i0;
        float *dxp = a.dx + (long long)n * a.C * HW + o00;
        const float *gp = a.dy + (long long)n * a.C * P + rem;
        for (int c = 0; c < a.C; c++) {
            const float g = ldg_stream(gp + (long long)c * P);
            float *q = dxp + (long long)c * HW;
            if (y0ok && x0ok) red_add(q, w00 * g);
            if (y0ok && x1ok) red_add(q + 1, w01 * g);
            if (y1ok && x0ok) red_add(q + a.W, w10 * g);
            if (y1ok && x1ok) red_add(q + a.W + 1, w11 * g);
        }
    }
}

int scatter_blocks_per_sample(long long P) {
    long long b = (P + kThreads - 1) / kThreads;
    return (int)(b > 4096 ? 4096 : b);
}

int dtheta_blocks_per_sample(int N, long long P) {
    long long by_pixels = (P + kThreads - 1) / kThreads;
    long long want = (8LL * kNumSMs + N - 1) / N;
    long long b = by_pixels < want ? by_pixels : want;
    return (int)(b < 1 ? 1 : b);
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace

size_t stn_ws_bytes(int N, int C, int H, int W, int Ho, int Wo) {
    (void)C;
    (void)H;
    (void)W;
    long long P = (long long)Ho * Wo;
    int bps = dtheta_blocks_per_sample(N, P);
    return align256(sizeof(double) * (size_t)N * bps * 6) + align256(sizeof(double) * Wo) +
           align256(sizeof(double) * Ho);
}

cudaError_t stn_fwd_launch(const StnArgs &a, cudaStream_t s) {
    long long total = (long long)a.N * a.Ho * a.Wo;
    unsigned blocks = (unsigned)((total + kThreads - 1) / kThreads);
    stn_fwd_kernel<<<blocks, kThreads, 0, s>>>(a);
    note_launch();
    return cudaGetLastError();
}

cudaError_t stn_bwd_launch(const StnArgs &a, int algo, int deterministic, void *ws,
                           size_t ws_bytes, cudaStream_t s) {
    (void)ws_bytes;
    (void)deterministic;
    const long long P = (long long)a.Ho * a.Wo;
    const int bps = dtheta_blocks_per_sample(a.N, P);
    char *w = (char *)ws;
    double *partials = (double *)w;
    w += align256(sizeof(double) * (size_t)a.N * bps * 6);
    double *xtab = (double *)w;
    w += align256(sizeof(double) * a.Wo);
    double *ytab = (double *)w;
    const int tmax = a.Wo > a.Ho ? a.Wo : a.Ho;
    stn_tables_kernel<<<(tmax + 255) / 256, 256, 0, s>>>(xtab, ytab, a.Ho, a.Wo, a.ac);
    note_launch();
    if (a.dtheta) {
        stn_dtheta_kernel<<<dim3(bps, a.N), kThreads, 0, s>>>(a, xtab, ytab, partials, bps);
        note_launch();
        stn_dtheta_finalize<<<a.N, kThreads, 0, s>>>(partials, bps, a.dtheta);
        note_launch();
    }
    if (a.dx) {
        // AUTO: gather (bounded affine preimage) unless border padding, where the clamp
        // has no bounded inverse (the API refuses deterministic=1 with border).
        const bool gather = (algo == 0 || algo == 1) && !a.border;
        const long long HW = (long long)a.H * a.W;
        if (gather) {
            unsigned blocks = (unsigned)(((long long)a.N * HW + kThreads - 1) / kThreads);
            if (a.C >= 16)
                stn_dx_gather_kernel<16><<<blocks, kThreads, 0, s>>>(a, xtab, ytab);
            else if (a.C >= 8)
                stn_dx_gather_kernel<8><<<blocks, kThreads, 0, s>>>(a, xtab, ytab);
            else
                stn_dx_gather_kernel<4><<<blocks, kThreads, 0, s>>>(a, xtab, ytab);
            note_launch();
            // samples whose theta is near-singular fall back to atomics
            stn_dx_scatter_kernel<<<dim3(scatter_blocks_per_sample(P), a.N), kThreads, 0, s>>>(a, 1);
            note_launch();
        } else {
            cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * HW, s);
            stn_dx_scatter_kernel<<<dim3(scatter_blocks_per_sample(P), a.N), kThreads, 0, s>>>(a, 0);
            note_launch();
        }
    }
    return cudaGetLastError();
}

}  // namespace rs
