// bslice.cu — HDRNet bilateral slice-apply, forward and adjoint, sm_100a.
//
// Geometry.  Pixel (y, x) sits at cell coordinates cx = (x+.5)Gw/W - .5,
// cy = (y+.5)Gh/H - .5 (R5).  A "dual cell" (j, k), j in [-1, Gh-1],
// k in [-1, Gw-1], is the set of pixels with floor(cy) = j and floor(cx) = k:
// every pixel of a dual cell reads the SAME four spatial grid corners
// (clamp(j+b), clamp(k+a)), b, a in {0,1}.  Blocks own a dual cell (or a
// sub-tile of a large one), so the block's grid footprint is 4 x D x 12
// coefficients staged once in shared memory (the "bounded footprint" of the
// scatter-to-gather conversion) and the per-pixel
// coefficients are applied on the fly, never materialised.
//
// Kernels
//   bslice_fwd_tiled      per pixel: 2-plane slice from smem corner lerps, apply.
//   bslice_bwd_tiled      per pixel: dX = A^T G, dguide = D G.(A_hi-A_lo)Xt, and
//                         d_grid accumulated WITHOUT atomics: pixels are
//                         counting-sorted by z-bin (floor(cz)) so a warp's 32
//                         lanes share the two z-planes; each lane keeps the 96
//                         (2 planes x 4 corners x 12 coeffs) sums in registers,
//                         reduce-scattered across the warp (93 shuffles) when
//                         the bin changes; per-warp smem slots are summed in
//                         fixed order into one partial per (dual cell, corner).
//   bslice_dgrid_gather   each grid cell sums its <=4 dual-cell partials in a
//                         fixed order (deterministic; the rfactor "partial +
//                         serial" split of PAPER.md:840).
//   bslice_*_generic      any shape: thread per pixel, grid via L1, d_grid by
//                         red.global.add (the atomic fallback).
#include "common.cuh"

namespace rs {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileX = 128;   // nominal max sub-tile width  (px)
constexpr int kTileY = 64;    // nominal max sub-tile height (px)
// a dual cell spans <= ceil(W/Gw) (+1 for fp rounding) pixels: smem holds +2 slack
constexpr int kTileXS = kTileX + 2, kTileYS = kTileY + 2;
constexpr int kPlaneStride = 13;  // float4 per z-plane in smem (12 + 1 pad: conflict-free)
constexpr unsigned kInvalid = 0xffffffffu;
constexpr int kChunk = 16;  // pixels per warp step in the backward (lane pairs)

// ----------------------------------------------------------------- exact coordinates (R5)
RS_DEV double bs_cx(int x, int W, int Gw) {
    return __dsub_rn(__ddiv_rn(__dmul_rn(__dadd_rn((double)x, 0.5), (double)Gw), (double)W), 0.5);
}

RS_DEV double bs_cz(float g, int D) { return __dsub_rn(__dmul_rn((double)g, (double)D), 0.5); }

RS_DEV int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// z-bin of a guide value: bin = clamp(floor(cz)+1, 0, D); planes (bin-1, bin) clamped.
RS_DEV void z_cell(float g, int D, int &bin, float &fz) {
    const double cz = bs_cz(g, D);
    const double fl = floor(cz);
    fz = (float)__dsub_rn(cz, fl);
    const double b = fl + 1.0;
    bin = b < 0.0 ? 0 : (b > (double)D ? D : (int)b);
    if (!(cz == cz)) { bin = 0; fz = 0.f; }  // NaN guide: defined, not meaningful
}

// first pixel index x with floor(cx(x)) >= k (exact, monotone search)
RS_DEV int dual_begin(int k, int W, int G) {
    if (k <= -1) return 0;
    if (k >= G) return W;
    int e = (int)ceil(((double)k + 0.5) * (double)W / (double)G - 0.5);
    e = clampi(e, 0, W);
    while (e > 0 && floor(bs_cx(e - 1, W, G)) >= (double)k) e--;
    while (e < W && floor(bs_cx(e, W, G)) < (double)k) e++;
    return e;
}

struct Tile {
    int n, j, k;         // sample, dual cell
    int ys, ye, xs, xe;  // pixel ranges [ys, ye) x [xs, xe)
};

// Block-wide tile descriptor: the four exact dual-cell bounds (fp64 searches with
// divisions) are computed once, by threads 0-3, and shared through `sh` (4 ints).
// Contains a __syncthreads: call from every thread of the block.
RS_DEV Tile tile_of_block(int b, int Gh, int Gw, int SY, int SX, int H, int W, int *sh) {
    Tile t;
    const int sx = b % SX;
    int bb = b / SX;
    const int sy = bb % SY;
    bb /= SY;
    const int kk = bb % (Gw + 1);
    bb /= (Gw + 1);
    const int jj = bb % (Gh + 1);
    t.n = bb / (Gh + 1);
    t.j = jj - 1;
    t.k = kk - 1;
    if (threadIdx.x < 4) {
        const int v = threadIdx.x;
        sh[v] = v < 2 ? dual_begin(t.j + v, H, Gh) : dual_begin(t.k + v - 2, W, Gw);
    }
    __syncthreads();
    const int yb = sh[0], yend = sh[1], xb = sh[2], xend = sh[3];
    const int hh = yend - yb, ww = xend - xb;
    t.ys = yb + (int)(((long long)hh * sy) / SY);
    t.ye = yb + (int)(((long long)hh * (sy + 1)) / SY);
    t.xs = xb + (int)(((long long)ww * sx) / SX);
    t.xe = xb + (int)(((long long)ww * (sx + 1)) / SX);
    return t;
}

RS_DEV Tile tile_of(int b, int Gh, int Gw, int SY, int SX, int H, int W) {
    Tile t;
    const int sx = b % SX;
    b /= SX;
    const int sy = b % SY;
    b /= SY;
    const int kk = b % (Gw + 1);
    b /= (Gw + 1);
    const int jj = b % (Gh + 1);
    t.n = b / (Gh + 1);
    t.j = jj - 1;
    t.k = kk - 1;
    const int yb = dual_begin(t.j, H, Gh), yend = dual_begin(t.j + 1, H, Gh);
    const int xb = dual_begin(t.k, W, Gw), xend = dual_begin(t.k + 1, W, Gw);
    const int hh = yend - yb, ww = xend - xb;
    t.ys = yb + (int)(((long long)hh * sy) / SY);
    t.ye = yb + (int)(((long long)hh * (sy + 1)) / SY);
    t.xs = xb + (int)(((long long)ww * sx) / SX);
    t.xe = xb + (int)(((long long)ww * (sx + 1)) / SX);
    return t;
}

// Dual-cell bounds table: tab[jj] = dual_begin(jj - 1, H, Gh) for jj in [0, Gh+1],
// tab[Gh + 2 + kk] = dual_begin(kk - 1, W, Gw) for kk in [0, Gw+1] (one tiny launch per
// backward call, so the tiles read their bounds instead of re-running fp64 searches).
__global__ void bslice_bounds_kernel(int *tab, int H, int W, int Gh, int Gw) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Gh + 2) tab[t] = dual_begin(t - 1, H, Gh);
    if (t < Gw + 2) tab[Gh + 2 + t] = dual_begin(t - 1, W, Gw);
}

RS_DEV Tile tile_of_tab(int b, int Gh, int Gw, int SY, int SX, const int *__restrict__ tab) {
    Tile t;
    const int sx = b % SX;
    b /= SX;
    const int sy = b % SY;
    b /= SY;
    const int kk = b % (Gw + 1);
    b /= (Gw + 1);
    const int jj = b % (Gh + 1);
    t.n = b / (Gh + 1);
    t.j = jj - 1;
    t.k = kk - 1;
    const int yb = __ldg(tab + jj), yend = __ldg(tab + jj + 1);
    const int xb = __ldg(tab + Gh + 2 + kk), xend = __ldg(tab + Gh + 2 + kk + 1);
    const int hh = yend - yb, ww = xend - xb;
    t.ys = yb + (int)(((long long)hh * sy) / SY);
    t.ye = yb + (int)(((long long)hh * (sy + 1)) / SY);
    t.xs = xb + (int)(((long long)ww * sx) / SX);
    t.xe = xb + (int)(((long long)ww * (sx + 1)) / SX);
    return t;
}

// Stage, for every z-bin b in [0, D] and coefficient q, the bilinear-lerp terms
// S(fx, fy) = a + fx b + fy (c + fx d) of (i) the low plane clamp(b-1) and (ii)
// the plane DIFFERENCE clamp(b) - clamp(b-1).  Slicing the difference directly
// (instead of subtracting two slices) keeps dA/dcz accurate to fp32 relative
// precision of the difference itself: it feeds d_guide (P3).
RS_DEV float4 lerp_terms(float c00, float c01, float c10, float c11) {
    return make_float4(c00, c01 - c00, c10 - c00, (c11 - c10) - (c01 - c00));
}

RS_DEV void stage_corners(float4 *glo, float4 *gdz, const float *grid, const Tile &t, int D,
                          int Gh, int Gw) {
    const int y0 = clampi(t.j, 0, Gh - 1), y1 = clampi(t.j + 1, 0, Gh - 1);
    const int x0 = clampi(t.k, 0, Gw - 1), x1 = clampi(t.k + 1, 0, Gw - 1);
    const long long plane = (long long)Gh * Gw;
    const float *g = grid + (long long)t.n * 12 * D * plane;
    for (int e = threadIdx.x; e < (D + 1) * 12; e += blockDim.x) {
        const int b = e / 12, q = e - b * 12;
        const int zl = clampi(b - 1, 0, D - 1), zh = clampi(b, 0, D - 1);
        const float *pl = g + ((long long)q * D + zl) * plane;
        const float *ph = g + ((long long)q * D + zh) * plane;
        const float l00 = __ldg(pl + y0 * Gw + x0), l01 = __ldg(pl + y0 * Gw + x1);
        const float l10 = __ldg(pl + y1 * Gw + x0), l11 = __ldg(pl + y1 * Gw + x1);
        const float h00 = __ldg(ph + y0 * Gw + x0), h01 = __ldg(ph + y0 * Gw + x1);
        const float h10 = __ldg(ph + y1 * Gw + x0), h11 = __ldg(ph + y1 * Gw + x1);
        glo[b * kPlaneStride + q] = lerp_terms(l00, l01, l10, l11);
        gdz[b * kPlaneStride + q] = lerp_terms(h00 - l00, h01 - l01, h10 - l10, h11 - l11);
    }
}

// Backward layout: per (bin, q) the low-plane and plane-difference lerp terms interleaved
// as float2 pairs {lo, dz}: gi[(b * kQS + q) * 2] = {a_lo, a_dz, b_lo, b_dz},
// gi[... + 1] = {c_lo, c_dz, d_lo, d_dz}, so one packed FMA (FFMA2) lerps both.
constexpr int kQS = 12;  // q per bin (the two float4 of a q are adjacent)
RS_DEV void stage_corners_i(float4 *gi, const float *grid, const Tile &t, int D, int Gh, int Gw) {
    const int y0 = clampi(t.j, 0, Gh - 1), y1 = clampi(t.j + 1, 0, Gh - 1);
    const int x0 = clampi(t.k, 0, Gw - 1), x1 = clampi(t.k + 1, 0, Gw - 1);
    const long long plane = (long long)Gh * Gw;
    const float *g = grid + (long long)t.n * 12 * D * plane;
    for (int e = threadIdx.x; e < (D + 1) * 12; e += blockDim.x) {
        const int b = e / 12, q = e - b * 12;
        const int zl = clampi(b - 1, 0, D - 1), zh = clampi(b, 0, D - 1);
        const float *pl = g + ((long long)q * D + zl) * plane;
        const float *ph = g + ((long long)q * D + zh) * plane;
        const float l00 = __ldg(pl + y0 * Gw + x0), l01 = __ldg(pl + y0 * Gw + x1);
        const float l10 = __ldg(pl + y1 * Gw + x0), l11 = __ldg(pl + y1 * Gw + x1);
        const float h00 = __ldg(ph + y0 * Gw + x0), h01 = __ldg(ph + y0 * Gw + x1);
        const float h10 = __ldg(ph + y1 * Gw + x0), h11 = __ldg(ph + y1 * Gw + x1);
        const float4 L = lerp_terms(l00, l01, l10, l11);
        const float4 Dz = lerp_terms(h00 - l00, h01 - l01, h10 - l10, h11 - l11);
        gi[(b * kQS + q) * 2] = make_float4(L.x, Dz.x, L.y, Dz.y);
        gi[(b * kQS + q) * 2 + 1] = make_float4(L.z, Dz.z, L.w, Dz.w);
    }
}

RS_DEV float2 f2(float a, float b) { return make_float2(a, b); }

RS_DEV float lerp2(const float4 c, float fx, float fy) {
    return fmaf(fy, fmaf(fx, c.w, c.z), fmaf(fx, c.y, c.x));
}

// ----------------------------------------------------------------- forward, tiled
__global__ void __launch_bounds__(kThreads)
    bslice_fwd_tiled(BsliceArgs a, int SY, int SX, int ntab) {
    extern __shared__ float4 smem4[];
    float4 *glo = smem4;                                       // (D+1) * 13
    float4 *gdz = glo + (a.D + 1) * kPlaneStride;              // (D+1) * 13
    float *fxt = (float *)(gdz + (a.D + 1) * kPlaneStride);    // kTileXS
    float *fyt = fxt + kTileXS;                                // kTileYS
    __shared__ int tsh[4];
    const Tile t = tile_of_block(blockIdx.x, a.Gh, a.Gw, SY, SX, a.H, a.W, tsh);
    const int TW = t.xe - t.xs, TH = t.ye - t.ys;
    if (TW <= 0 || TH <= 0) return;
    stage_corners(glo, gdz, a.grid, t, a.D, a.Gh, a.Gw);
    for (int c = threadIdx.x; c < TW; c += kThreads) {
        const double cx = bs_cx(t.xs + c, a.W, a.Gw);
        fxt[c] = (float)__dsub_rn(cx, floor(cx));
    }
    for (int r = threadIdx.x; r < TH; r += kThreads) {
        const double cy = bs_cx(t.ys + r, a.H, a.Gh);
        fyt[r] = (float)__dsub_rn(cy, floor(cy));
    }
    __syncthreads();
    const long long HW = (long long)a.H * a.W;
    const float *gd = a.guide + (long long)t.n * HW;
    const float *xp = a.x + (long long)t.n * 3 * HW;
    float *yp = a.y + (long long)t.n * 3 * HW;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int NB = a.D + 1;
    // per-warp row table: for the current row's fy, (a + fy c, b + fy d) of the low
    // plane and of the plane difference, for every (bin, q), bins kPlaneStride float4
    // apart (conflict-free across bins): one LDS.128 per coefficient and pixel
    float4 *rt = (float4 *)(fyt + kTileYS) + w * ntab * kPlaneStride * NB;  // ntab (1 or 2) tables per warp
    // the warp's items, two pixels per lane: (row r, 64-column segment cx) -- or, for a dual
    // cell at most 32 px wide, rows r and r + kWarps at column lane (a second row table),
    // so both pixels are live; the next item's guide and X loads are issued before the
    // current item is computed (a small dual cell has one item per row: without the
    // prefetch every row waits a round trip)
    const bool pairs = ntab == 2 && TW <= 32;
    const int ncx = pairs ? 1 : (TW + 63) >> 6;
    auto row_of = [&](int r, int k) { return pairs ? r + k * kWarps : r; };
    auto col_of = [&](int cx, int k) { return pairs ? lane : cx * 64 + lane + 32 * k; };
    float gn[2] = {0.f, 0.f}, xn[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    auto fetch = [&](int r, int cx) {
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int rk = row_of(r, k), c = col_of(cx, k);
            const bool ok = rk < TH && c < TW;
            const long long o = ok ? (long long)(t.ys + rk) * a.W + t.xs + c : 0;
            gn[k] = ok ? ldg_stream(gd + o) : 0.f;
#pragma unroll
            for (int i = 0; i < 3; i++) xn[k][i] = ok ? ldg_stream(xp + i * HW + o) : 0.f;
        }
    };
    const int rstep = pairs ? 2 * kWarps : kWarps;
    fetch(w, 0);
    int r = w, cx = 0;
    while (r < TH) {
        float gv[2], xv[2][3];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            gv[k] = gn[k];
#pragma unroll
            for (int i = 0; i < 3; i++) xv[k][i] = xn[k][i];
        }
        const int cx1 = cx + 1 < ncx ? cx + 1 : 0, r1 = cx + 1 < ncx ? r : r + rstep;
        fetch(r1, cx1);
        if (cx == 0) {
            // per-warp row table(s): for the row's fy, (a + fy c, b + fy d) of the low plane
            // and of the plane difference, for every (bin, q), bins kPlaneStride float4
            // apart (conflict-free across bins): one LDS.128 per coefficient and pixel
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (k == 1 && !(pairs && r + kWarps < TH)) break;
                const float fy = fyt[row_of(r, k)];
                float4 *tk = rt + k * kPlaneStride * NB;
                for (int e = lane; e < 12 * NB; e += 32) {
                    const int b = e / 12, q = e - b * 12;
                    const float4 L = glo[b * kPlaneStride + q], Dz = gdz[b * kPlaneStride + q];
                    tk[b * kPlaneStride + q] = make_float4(fmaf(fy, L.z, L.x), fmaf(fy, L.w, L.y),
                                                           fmaf(fy, Dz.z, Dz.x), fmaf(fy, Dz.w, Dz.y));
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int rk = row_of(r, k), c = col_of(cx, k);
            if (rk >= TH || c >= TW) continue;
            const long long o = (long long)(t.ys + rk) * a.W + t.xs + c;
            const float fx = fxt[c];
            int bin;
            float fz;
            z_cell(gv[k], a.D, bin, fz);
            const float4 *T = rt + (pairs ? k : 0) * kPlaneStride * NB + bin * kPlaneStride;
#pragma unroll
            for (int oc = 0; oc < 3; oc++) {
                float A[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float4 v = T[4 * oc + i];
                    A[i] = fmaf(fz, fmaf(fx, v.w, v.z), fmaf(fx, v.y, v.x));
                }
                yp[oc * HW + o] = fmaf(A[0], xv[k][0], fmaf(A[1], xv[k][1], fmaf(A[2], xv[k][2], A[3])));
            }
        }
        r = r1;
        cx = cx1;
    }
}

// ----------------------------------------------------------------- backward, tiled
// 96-vector reduce-scatter across the warp: after it lane holds 3 sums for
// indices base .. base+2, base = 48 b4 + 24 b3 + 12 b2 + 6 b1 + 3 b0.
template <int H>
RS_DEV void rs_stage(float *v, int lane, int m) {
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int k = 0; k < H; k++) {
        const float send = hi ? v[k] : v[k + H];
        const float keep = hi ? v[k + H] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
}

// Lane pairs: lane 2s+e owns pixel slot s of the chunk and coefficient half e
// (q = 6e .. 6e+5) of BOTH z-planes.  acc index: (p*4 + corner)*6 + qq, p = plane
// (0: clamp(bin-1), 1: clamp(bin)), corner = b*2 + a (spatial), q = 6e + qq.
// Reduce-scatter across the 16 lanes of the same half (xor 16, 8, 4, 2: 45
// shuffles); lane then owns 3 sums, base = 24 b4 + 12 b3 + 6 b2 + 3 b1.
// wacc (warp slot): [corner(4)][z(D)][q(12)]
// kQmap: false -> lane e holds q = 6e + qq; true (split kernel) -> q = 4e + qq (qq < 4),
// 8 + 2e + (qq - 4) (qq >= 4): both halves then read G and Xt in the same pattern
template <bool kQmap = false>
RS_DEV void flush_acc(float *acc, float *wacc, int bin, int D, int lane) {
    rs_stage<24>(acc, lane, 16);
    rs_stage<12>(acc, lane, 8);
    rs_stage<6>(acc, lane, 4);
    rs_stage<3>(acc, lane, 2);
    const int base = ((lane & 16) ? 24 : 0) + ((lane & 8) ? 12 : 0) + ((lane & 4) ? 6 : 0) + ((lane & 2) ? 3 : 0);
    const int e = lane & 1, p = (lane >> 4) & 1;
    const int z = p ? clampi(bin, 0, D - 1) : clampi(bin - 1, 0, D - 1);
    // plane-0 lanes first, then plane-1: the two planes coincide when clamped
#pragma unroll
    for (int ph = 0; ph < 2; ph++) {
        if (p == ph) {
#pragma unroll
            for (int t = 0; t < 3; t++) {
                const int idx = (base + t) % 24;  // (corner, qq) within the plane
                const int qq = idx % 6, corner = idx / 6;
                const int q = kQmap ? (qq < 4 ? 4 * e + qq : 8 + 2 * e + (qq - 4)) : 6 * e + qq;
                wacc[(corner * D + z) * 12 + q] += acc[t];
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 48; k++) acc[k] = 0.f;
}

__global__ void __launch_bounds__(kThreads, 2)
    bslice_bwd_tiled(BsliceArgs a, int SY, int SX, float *__restrict__ partials, const int *__restrict__ tab) {
    extern __shared__ float4 smem4[];
    const int D = a.D, NB = D + 1;
    float4 *gi = smem4;                                     // (D+1)*12*2 float4 (interleaved lo/dz)
    float *fxt = (float *)(gi + 2 * (D + 1) * kPlaneStride);  // kTileXS
    float *fyt = fxt + kTileXS;                             // kTileYS
    float *wacc = fyt + kTileYS;                            // kWarps * 4 * D * 12
    int *cnt = (int *)(wacc + kWarps * 4 * D * 12);         // kWarps * NB
    int *bstart = cnt + kWarps * NB;                        // NB + 1
    int *chunk_bin = bstart + NB + 1;                       // max chunks
    const int max_chunks = (kTileXS * kTileYS) / kChunk + 1 + NB;
    unsigned *sorted = (unsigned *)(chunk_bin + max_chunks);  // max_chunks * kChunk
    float *fzv = (float *)(((uintptr_t)(sorted + max_chunks * kChunk) + 15) & ~(uintptr_t)15);  // kTileXS*kTileYS
    unsigned char *binv = (unsigned char *)(fzv + kTileXS * kTileYS);    // kTileXS*kTileYS

    const Tile t = tile_of_tab(blockIdx.x, a.Gh, a.Gw, SY, SX, tab);
    const int TW = t.xe - t.xs, TH = t.ye - t.ys;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long HW = (long long)a.H * a.W;
    const float *gd = a.guide + (long long)t.n * HW;

    // guide tile -> smem (cp.async; overlaps the corner staging below)
    {
        const bool vec = (TW % 4 == 0) && (a.W % 4 == 0) && (t.xs % 4 == 0) &&
                         (((uintptr_t)a.guide & 15u) == 0);
        const int wq = vec ? TW / 4 : TW;
        for (int e = threadIdx.x; e < TH * wq; e += kThreads) {
            const int r = e / wq, q = e - r * wq;
            const float *src = gd + (long long)(t.ys + r) * a.W + t.xs;
            if (vec) cp_async16(fzv + r * TW + 4 * q, src + 4 * q);
            else cp_async4(fzv + r * TW + q, src + q);
        }
        cp_async_commit();
    }

    stage_corners_i(gi, a.grid, t, D, a.Gh, a.Gw);
    for (int c = threadIdx.x; c < TW; c += kThreads) {
        const double cx = bs_cx(t.xs + c, a.W, a.Gw);
        fxt[c] = (float)__dsub_rn(cx, floor(cx));
    }
    for (int r = threadIdx.x; r < TH; r += kThreads) {
        const double cy = bs_cx(t.ys + r, a.H, a.Gh);
        fyt[r] = (float)__dsub_rn(cy, floor(cy));
    }
    for (int e = threadIdx.x; e < kWarps * 4 * D * 12; e += kThreads) wacc[e] = 0.f;
    for (int e = threadIdx.x; e < kWarps * NB; e += kThreads) cnt[e] = 0;
    cp_async_wait<0>();
    __syncthreads();

    // ---- pass A: z-bin of every pixel, per-warp counts (warp w: rows w, w+8, ...)
    for (int r = w; r < TH; r += kWarps) {
        for (int c0 = 0; c0 < TW; c0 += 32) {
            const int c = c0 + lane;
            int bin = -1;
            if (c < TW) {
                float fz;
                z_cell(fzv[r * TW + c], D, bin, fz);  // guide value staged above, fz in place
                binv[r * TW + c] = (unsigned char)bin;
                fzv[r * TW + c] = fz;
            }
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(m) - 1) cnt[w * NB + bin] += __popc(m);
            __syncwarp();  // the next iteration's leader may update the same counter
        }
    }
    __syncthreads();
    // ---- scan: bin segments padded to kChunk, per-(warp, bin) offsets (warp 0: lane = bin,
    // a warp-wide exclusive scan of the padded bin sizes; the same offsets as a serial
    // bin-major / warp-minor walk)
    if (threadIdx.x < 32) {
        const int lane0 = threadIdx.x;
        int run = 0;
        for (int base = 0; base < NB; base += 32) {
            const int b = base + lane0;
            int tot = 0;
            if (b < NB)
                for (int ww = 0; ww < kWarps; ww++) tot += cnt[ww * NB + b];
            const int padded = (tot + kChunk - 1) & ~(kChunk - 1);
            int v = padded;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t2 = __shfl_up_sync(0xffffffffu, v, o);
                if (lane0 >= o) v += t2;
            }
            if (b < NB) {
                int off = run + v - padded;
                bstart[b] = off;
                for (int ww = 0; ww < kWarps; ww++) {
                    const int c2 = cnt[ww * NB + b];
                    cnt[ww * NB + b] = off;
                    off += c2;
                }
            }
            run += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane0 == 0) bstart[NB] = run;
    }
    __syncthreads();
    const int L = bstart[NB], nchunks = L / kChunk;
    for (int e = threadIdx.x; e < L; e += kThreads) sorted[e] = kInvalid;
    for (int c = threadIdx.x; c < nchunks; c += kThreads) {
        int b = 0;
        while (bstart[b + 1] <= c * kChunk) b++;
        chunk_bin[c] = b;
    }
    __syncthreads();
    // ---- pass B: stable placement (same walk order as pass A)
    for (int r = w; r < TH; r += kWarps) {
        for (int c0 = 0; c0 < TW; c0 += 32) {
            const int c = c0 + lane;
            const int bin = (c < TW) ? (int)binv[r * TW + c] : -1;
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0) {
                const int rank = __popc(m & ((1u << lane) - 1u));
                sorted[cnt[w * NB + bin] + rank] = ((unsigned)r << 16) | (unsigned)c;
            }
            __syncwarp();
            if (bin >= 0 && lane == __ffs(m) - 1) cnt[w * NB + bin] += __popc(m);
            __syncwarp();
        }
    }
    __syncthreads();

    // ---- pass C: per-chunk work, warp w takes a contiguous chunk range
    const float *xp = a.x + (long long)t.n * 3 * HW;
    const float *gp = a.dy + (long long)t.n * 3 * HW;
    float *dxp = a.dx ? a.dx + (long long)t.n * 3 * HW : nullptr;
    float *dgp = a.dguide ? a.dguide + (long long)t.n * HW : nullptr;
    float *mywacc = wacc + w * 4 * D * 12;
    const int cbeg = (int)(((long long)nchunks * w) / kWarps);
    const int cend = (int)(((long long)nchunks * (w + 1)) / kWarps);
    // acc2[(pl * 2 + bb) * 6 + qq] = the (corner a = 0, a = 1) pair of plane pl, corner
    // row bb, coefficient 6 e + qq: the 48 sums of flush_acc's layout as 24 float2 so the
    // trilinear-weighted updates are packed FMAs (FFMA2)
    float2 acc2[24];
#pragma unroll
    for (int k = 0; k < 24; k++) acc2[k] = f2(0.f, 0.f);
    auto flush2 = [&](int bin) {
        float acc[48];
#pragma unroll
        for (int pl = 0; pl < 2; pl++)
#pragma unroll
            for (int bb = 0; bb < 2; bb++)
#pragma unroll
                for (int qq = 0; qq < 6; qq++) {
                    acc[(pl * 4 + bb * 2 + 0) * 6 + qq] = acc2[(pl * 2 + bb) * 6 + qq].x;
                    acc[(pl * 4 + bb * 2 + 1) * 6 + qq] = acc2[(pl * 2 + bb) * 6 + qq].y;
                }
        flush_acc(acc, mywacc, bin, D, lane);
#pragma unroll
        for (int k = 0; k < 24; k++) acc2[k] = f2(0.f, 0.f);
    };
    const int slot = lane >> 1, e_pl = lane & 1;
    int cur_bin = cbeg < cend ? chunk_bin[cbeg] : 0;
    // software pipeline, distance 2: chunk ch+2's X / dY loads are issued while ch computes
    unsigned ent_a = cbeg < cend ? sorted[cbeg * kChunk + slot] : kInvalid;
    unsigned ent_b = cbeg + 1 < cend ? sorted[(cbeg + 1) * kChunk + slot] : kInvalid;
    float Xa[3] = {0.f, 0.f, 0.f}, Ga[3] = {0.f, 0.f, 0.f}, Xb[3] = {0.f, 0.f, 0.f}, Gb[3] = {0.f, 0.f, 0.f};
    auto fetch = [&](unsigned ent, float *Xd, float *Gd) {
        if (ent != kInvalid) {
            const long long o = (long long)(t.ys + (int)(ent >> 16)) * a.W + t.xs + (int)(ent & 0xffffu);
#pragma unroll
            for (int i = 0; i < 3; i++) {
                Xd[i] = __ldg(xp + i * HW + o);
                Gd[i] = __ldg(gp + i * HW + o);
            }
        }
    };
    fetch(ent_a, Xa, Ga);
    fetch(ent_b, Xb, Gb);
    for (int ch = cbeg; ch < cend; ch++) {
        const int bin = chunk_bin[ch];
        if (bin != cur_bin) {
            flush2(cur_bin);
            cur_bin = bin;
        }
        const unsigned ent = ent_a;
        float X[3], G[3];
#pragma unroll
        for (int i = 0; i < 3; i++) { X[i] = Xa[i]; G[i] = Ga[i]; Xa[i] = Xb[i]; Ga[i] = Gb[i]; }
        ent_a = ent_b;
        if (ch + 2 < cend) {
            ent_b = sorted[(ch + 2) * kChunk + slot];
            fetch(ent_b, Xb, Gb);
        }
        const bool valid = ent != kInvalid;
        const int r = valid ? (int)(ent >> 16) : 0, c = valid ? (int)(ent & 0xffffu) : 0;
        const long long o = (long long)(t.ys + r) * a.W + t.xs + c;
        const float fx = fxt[c], fy = fyt[r];
        const float fz = valid ? fzv[r * TW + c] : 0.f;
        if (!valid) {
#pragma unroll
            for (int i = 0; i < 3; i++) { X[i] = 0.f; G[i] = 0.f; }
        }
        // this lane's coefficient half: q = 6 e + qq, (oc, i) = (q / 4, q % 4)
        const float4 *Qc = gi + (bin * kQS + 6 * e_pl) * 2;
        const bool e1 = e_pl != 0;
        const float Gq[6] = {e1 ? G[1] : G[0], e1 ? G[1] : G[0], e1 ? G[2] : G[0],
                             e1 ? G[2] : G[0], e1 ? G[2] : G[1], e1 ? G[2] : G[1]};
        const float Xq[6] = {e1 ? X[2] : X[0], e1 ? 1.f : X[1], e1 ? X[0] : X[2],
                             e1 ? X[1] : 1.f, e1 ? X[2] : X[0], e1 ? 1.f : X[1]};
        float2 wt2[4];  // (plane, corner row) x (corner a = 0, 1) trilinear weights
        {
            const float2 wx2 = f2(1.f - fx, fx);
            const float wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
#pragma unroll
            for (int pl = 0; pl < 2; pl++)
#pragma unroll
                for (int bb = 0; bb < 2; bb++) {
                    const float wzy = wz[pl] * wy[bb];
                    wt2[pl * 2 + bb] = __fmul2_rn(f2(wzy, wzy), wx2);
                }
        }
        const float2 fx2 = f2(fx, fx), fy2 = f2(fy, fy);
        float u[4] = {0.f, 0.f, 0.f, 0.f}, dgd = 0.f;
#pragma unroll
        for (int qq = 0; qq < 6; qq++) {
            const float4 v0 = Qc[2 * qq], v1 = Qc[2 * qq + 1];
            // {lo, d} = fy (fx w + z) + (fx y + x) for the low plane and the difference
            const float2 th = __ffma2_rn(fx2, f2(v1.z, v1.w), f2(v1.x, v1.y));
            const float2 tl = __ffma2_rn(fx2, f2(v0.z, v0.w), f2(v0.x, v0.y));
            const float2 ld = __ffma2_rn(fy2, th, tl);
            const float lo = ld.x, d = ld.y;
            const float P = Gq[qq] * Xq[qq];
            u[qq & 3] = fmaf(Gq[qq], fmaf(fz, d, lo), u[qq & 3]);  // A_q G_oc (i = 3 slots unused)
            dgd = fmaf(P, d, dgd);
            const float2 P2 = f2(P, P);
#pragma unroll
            for (int k = 0; k < 4; k++) acc2[k * 6 + qq] = __ffma2_rn(wt2[k], P2, acc2[k * 6 + qq]);
        }
        // dX_i = sum_oc A_{4oc+i} G_oc: this half's slots, then the partner's half
        float dx0 = e1 ? u[2] : u[0], dx1 = e1 ? u[3] : u[1], dx2 = e1 ? u[0] : u[2];
        dx0 += __shfl_xor_sync(0xffffffffu, dx0, 1);
        dx1 += __shfl_xor_sync(0xffffffffu, dx1, 1);
        dx2 += __shfl_xor_sync(0xffffffffu, dx2, 1);
        dgd += __shfl_xor_sync(0xffffffffu, dgd, 1);
        if (valid) {
            if (e_pl == 0) {
                if (dxp) {
                    dxp[o] = dx0;
                    dxp[HW + o] = dx1;
                }
            } else {
                if (dxp) dxp[2 * HW + o] = dx2;
                if (dgp) dgp[o] = (float)D * dgd;
            }
        }
    }
    if (cbeg < cend) flush2(cur_bin);
    __syncthreads();
    // ---- block partial: fixed-order sum over warps
    float *part = partials + (long long)blockIdx.x * 4 * D * 12;
    for (int e = threadIdx.x; e < 4 * D * 12; e += kThreads) {
        float s = 0.f;
#pragma unroll
        for (int ww = 0; ww < kWarps; ww++) s += wacc[ww * 4 * D * 12 + e];
        part[e] = s;
    }
}

// ----------------------------------------------------------------- backward, split phases
// bslice_bwd_split: the same dual-cell ownership, z-bin counting sort and lane-pair
// register accumulation of d_grid as bslice_bwd_tiled, with the per-pixel work moved
// out of the accumulation loop:
//   phase 1 (lane = pixel, raster order, coalesced 32-bit-offset loads and stores):
//           slice A (12 coefficients, both planes), dX = A^T G and d_guide, and the
//           pixel's record {G, X, fz, (r, c)} written to its bin-sorted slot in shared
//           memory (the stable counting-sort placement);
//   phase 2 (lane pairs over 16-record chunks of one bin): only the 96 trilinear-
//           weighted products P_q = G_oc Xt_i per pixel into register sums, flushed by
//           the same reduce-scatter as bslice_bwd_tiled, one partial per (tile, corner).
// Sub-tiles are at most kV2TX x kV2TY px so two blocks fit per SM.  (PAPER.md:36-42
// slice-apply; PAPER.md:700-731 bounded-footprint gather for d_grid.)
#ifndef RS_V2TY
#define RS_V2TY 32
#endif
#ifndef RS_V2MINB
#define RS_V2MINB 2
#endif
constexpr int kV2TX = 64, kV2TY = RS_V2TY;            // nominal max sub-tile (px)
constexpr int kV2PX = (kV2TX + 2) * (kV2TY + 2);      // per-tile pixel capacity (+1 rounding slack per axis)
constexpr int kBinS = 25;                             // float4 per bin in gi (24 + 1: lanes on different bins hit different banks)

RS_DEV int v2_maxch(int NB) { return kV2PX / kChunk + NB + 1; }

RS_DEV void stage_corners_b(float4 *gi, const float *grid, const Tile &t, int D, int Gh, int Gw) {
    const int y0 = clampi(t.j, 0, Gh - 1), y1 = clampi(t.j + 1, 0, Gh - 1);
    const int x0 = clampi(t.k, 0, Gw - 1), x1 = clampi(t.k + 1, 0, Gw - 1);
    const long long plane = (long long)Gh * Gw;
    const float *g = grid + (long long)t.n * 12 * D * plane;
    for (int e = threadIdx.x; e < (D + 1) * 12; e += blockDim.x) {
        const int b = e / 12, q = e - b * 12;
        const int zl = clampi(b - 1, 0, D - 1), zh = clampi(b, 0, D - 1);
        const float *pl = g + ((long long)q * D + zl) * plane;
        const float *ph = g + ((long long)q * D + zh) * plane;
        const float l00 = __ldg(pl + y0 * Gw + x0), l01 = __ldg(pl + y0 * Gw + x1);
        const float l10 = __ldg(pl + y1 * Gw + x0), l11 = __ldg(pl + y1 * Gw + x1);
        const float h00 = __ldg(ph + y0 * Gw + x0), h01 = __ldg(ph + y0 * Gw + x1);
        const float h10 = __ldg(ph + y1 * Gw + x0), h11 = __ldg(ph + y1 * Gw + x1);
        const float4 L = lerp_terms(l00, l01, l10, l11);
        const float4 Dz = lerp_terms(h00 - l00, h01 - l01, h10 - l10, h11 - l11);
        gi[b * kBinS + 2 * q] = make_float4(L.x, Dz.x, L.y, Dz.y);
        gi[b * kBinS + 2 * q + 1] = make_float4(L.z, Dz.z, L.w, Dz.w);
    }
}

// NW warps per block; CAP pixels of record capacity (NW = 4: cells of at most 33 x 33 px)
template <bool kMulti, int NW = 8>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? 4 : RS_V2MINB)
    bslice_bwd_split(BsliceArgs a, int SY, int SX, float *__restrict__ partials, const int *__restrict__ tab) {
    extern __shared__ float4 smem4[];
    const int D = a.D, NB = D + 1;
    constexpr int kNT = NW * 32, CAP = NW == 4 ? 34 * 34 : kV2PX;
    const int maxch = CAP / kChunk + NB + 1;
    float4 *rec = smem4;                                   // maxch * kChunk * 2 (32-B records)
    float4 *gi = rec + maxch * kChunk * 2;                 // NB * kBinS
    float *fzv = (float *)(gi + NB * kBinS);               // CAP: guide, then fz in place
    float *fxt = fzv + CAP;                              // kV2TX + 4
    float *fyt = fxt + kV2TX + 4;                          // kV2TY + 4
    float *wacc = fyt + kV2TY + 4;                         // NW * 4 * D * 12
    int *cnt = (int *)(wacc + NW * 4 * D * 12);        // NW * NB
    int *bstart = cnt + NW * NB;                       // NB + 1
    int *chunk_bin = bstart + NB + 1;                      // maxch
    unsigned char *binv = (unsigned char *)(chunk_bin + maxch);  // CAP

    // the block owns a whole dual cell (column split SX); its rows are walked as
    // sub-tiles of <= kV2TY rows (the records hold 32 B per pixel)
    __shared__ int tsh[4];  // (tab == nullptr: the block searches its dual cell's bounds itself)
    const Tile tc = tab ? tile_of_tab(blockIdx.x, a.Gh, a.Gw, SY, SX, tab)
                        : tile_of_block(blockIdx.x, a.Gh, a.Gw, SY, SX, a.H, a.W, tsh);
    const int TW = tc.xe - tc.xs, THc = tc.ye - tc.ys;
    const int nsub = (THc + kV2TY - 1) / kV2TY;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long HW = (long long)a.H * a.W;
    stage_corners_b(gi, a.grid, tc, D, a.Gh, a.Gw);
    for (int c = threadIdx.x; c < TW; c += kNT) {
        const double cx = bs_cx(tc.xs + c, a.W, a.Gw);
        fxt[c] = (float)__dsub_rn(cx, floor(cx));
    }
    for (int e = threadIdx.x; e < NW * 4 * D * 12; e += kNT) wacc[e] = 0.f;
    float *mywacc = wacc + w * 4 * D * 12;
    float2 acc2[24];
#pragma unroll
    for (int k = 0; k < 24; k++) acc2[k] = f2(0.f, 0.f);
    auto flush2 = [&](int bin) {
        float acc[48];
#pragma unroll
        for (int pl = 0; pl < 2; pl++)
#pragma unroll
            for (int bb = 0; bb < 2; bb++)
#pragma unroll
                for (int qq = 0; qq < 6; qq++) {
                    acc[(pl * 4 + bb * 2 + 0) * 6 + qq] = acc2[(pl * 2 + bb) * 6 + qq].x;
                    acc[(pl * 4 + bb * 2 + 1) * 6 + qq] = acc2[(pl * 2 + bb) * 6 + qq].y;
                }
        flush_acc<true>(acc, mywacc, bin, D, lane);
#pragma unroll
        for (int k = 0; k < 24; k++) acc2[k] = f2(0.f, 0.f);
    };
    const int slot = lane >> 1;
    const bool e1 = (lane & 1) != 0;
    int cur_bin = -1;  // bin of the pending register sums (-1: none)
    for (int sub = 0; sub < nsub; sub++) {
    Tile t = tc;
    t.ys = tc.ys + (int)(((long long)THc * sub) / nsub);
    t.ye = tc.ys + (int)(((long long)THc * (sub + 1)) / nsub);
    const int TH = t.ye - t.ys;
    const long long tbase = (long long)t.ys * a.W + t.xs;  // tile origin within a plane
    __syncthreads();  // the previous sub-tile's records, bins and counts are consumed
    {  // guide tile -> smem (cp.async; overlaps the corner staging below)
        const float *gd = a.guide + (long long)t.n * HW + tbase;
        const bool vec = (TW % 4 == 0) && (a.W % 4 == 0) && (t.xs % 4 == 0) && (((uintptr_t)a.guide & 15u) == 0);
        const int wq = vec ? TW / 4 : TW;
        for (int e = threadIdx.x; e < TH * wq; e += kNT) {
            const int r = e / wq, q = e - r * wq;
            const float *src = gd + (long long)r * a.W;
            if (vec) cp_async16(fzv + r * TW + 4 * q, src + 4 * q);
            else cp_async4(fzv + r * TW + q, src + q);
        }
        cp_async_commit();
    }
    for (int r = threadIdx.x; r < TH; r += kNT) {
        const double cy = bs_cx(t.ys + r, a.H, a.Gh);
        fyt[r] = (float)__dsub_rn(cy, floor(cy));
    }
    for (int e = threadIdx.x; e < NW * NB; e += kNT) cnt[e] = 0;
    cp_async_wait<0>();
    __syncthreads();

    // ---- phase 0: z-bin of every pixel, per-warp counts (warp w: rows w, w+8, ...)
    for (int r = w; r < TH; r += NW) {
        for (int c0 = 0; c0 < TW; c0 += 32) {
            const int c = c0 + lane;
            int bin = -1;
            if (c < TW) {
                float fz;
                z_cell(fzv[r * TW + c], D, bin, fz);
                binv[r * TW + c] = (unsigned char)bin;
                fzv[r * TW + c] = fz;
            }
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(m) - 1) cnt[w * NB + bin] += __popc(m);
            __syncwarp();
        }
    }
    __syncthreads();
    // ---- scan (warp 0, lane = bin): bin segments padded to kChunk, per-(warp, bin)
    // offsets; the padding slots get zero records (G = X = 0: no contribution)
    if (threadIdx.x < 32) {
        int run = 0;
        for (int base = 0; base < NB; base += 32) {
            const int b = base + lane;
            int tot = 0;
            if (b < NB)
                for (int ww = 0; ww < NW; ww++) tot += cnt[ww * NB + b];
            const int padded = (tot + kChunk - 1) & ~(kChunk - 1);
            int v = padded;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t2 = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t2;
            }
            if (b < NB) {
                int off = run + v - padded;
                bstart[b] = off;
                for (int ww = 0; ww < NW; ww++) {
                    const int c2 = cnt[ww * NB + b];
                    cnt[ww * NB + b] = off;
                    off += c2;
                }
                for (int e = off; e < run + v; e++) {
                    rec[2 * e] = make_float4(0.f, 0.f, 0.f, 0.f);
                    rec[2 * e + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            run += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) bstart[NB] = run;
    }
    __syncthreads();
    const int nchunks = bstart[NB] / kChunk;
    for (int c = threadIdx.x; c < nchunks; c += kNT) {
        int b = 0;
        while (bstart[b + 1] <= c * kChunk) b++;
        chunk_bin[c] = b;
    }

    // ---- phase 1: lane = pixel (same walk order as phase 0: stable placement)
    {
        const long long nb3 = (long long)t.n * 3 * HW + tbase;
        const float *x0p = a.x + nb3, *x1p = x0p + HW, *x2p = x1p + HW;
        const float *g0p = a.dy + nb3, *g1p = g0p + HW, *g2p = g1p + HW;
        float *d0p = a.dx ? a.dx + nb3 : nullptr;
        float *dgp = a.dguide ? a.dguide + (long long)t.n * HW + tbase : nullptr;
        const float Df = (float)D;
        // the warp's (row, 32-column segment) items in phase-0 order; the next item's six
        // global loads are issued before the current one is processed (pipeline depth 1)
        const int ncx = (TW + 31) >> 5;
        float Xn[3] = {0.f, 0.f, 0.f}, Gn[3] = {0.f, 0.f, 0.f};
        auto fetch = [&](int r, int c) {
            if (r < TH && c < TW) {
                const int o = r * a.W + c;
                Xn[0] = ldg_stream(x0p + o); Xn[1] = ldg_stream(x1p + o); Xn[2] = ldg_stream(x2p + o);
                Gn[0] = ldg_stream(g0p + o); Gn[1] = ldg_stream(g1p + o); Gn[2] = ldg_stream(g2p + o);
            }
        };
        fetch(w, lane);
        int r = w, cx = 0;
        while (r < TH) {
            const int c = cx * 32 + lane;
            float X[3], G[3];
#pragma unroll
            for (int i = 0; i < 3; i++) { X[i] = Xn[i]; G[i] = Gn[i]; }
            const int cx1 = cx + 1 < ncx ? cx + 1 : 0, r1 = cx + 1 < ncx ? r : r + NW;
            fetch(r1, cx1 * 32 + lane);
            const bool ok = c < TW;
            const int o = r * a.W + c;
            const float2 fy2 = f2(fyt[r], fyt[r]);
            const int bin = ok ? (int)binv[r * TW + c] : -1;
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (ok) {
                const float fz = fzv[r * TW + c];
                const float fx = fxt[c];
                const float2 fx2 = f2(fx, fx);
                const float4 *Qb = gi + bin * kBinS;
                float A[12], dq[12];
#pragma unroll
                for (int q = 0; q < 12; q++) {
                    const float4 v0 = Qb[2 * q], v1 = Qb[2 * q + 1];
                    const float2 th = __ffma2_rn(fx2, f2(v1.z, v1.w), f2(v1.x, v1.y));
                    const float2 tl = __ffma2_rn(fx2, f2(v0.z, v0.w), f2(v0.x, v0.y));
                    const float2 ld = __ffma2_rn(fy2, th, tl);
                    A[q] = fmaf(fz, ld.y, ld.x);
                    dq[q] = ld.y;
                }
                // dX_i = sum_oc A_{4 oc + i} G_oc, d_guide = D sum_q G_oc Xt_i dA_q/dz
                // (the summation order of bslice_bwd_tiled's lane pairs)
                const float Xt[4] = {X[0], X[1], X[2], 1.f};
                float dlo = 0.f, dhi = 0.f;
#pragma unroll
                for (int q = 0; q < 6; q++) dlo = fmaf(G[q >> 2] * Xt[q & 3], dq[q], dlo);
#pragma unroll
                for (int q = 6; q < 12; q++) dhi = fmaf(G[q >> 2] * Xt[q & 3], dq[q], dhi);
                if (d0p) {
                    // (explicit _rn: no contraction of the final sums into FMAs)
                    const float dx0 = __fadd_rn(fmaf(G[1], A[4], fmaf(G[0], A[0], 0.f)), __fmul_rn(G[2], A[8]));
                    const float dx1 = __fadd_rn(fmaf(G[1], A[5], fmaf(G[0], A[1], 0.f)), __fmul_rn(G[2], A[9]));
                    const float dx2 = __fadd_rn(__fmul_rn(G[0], A[2]), fmaf(G[2], A[10], fmaf(G[1], A[6], 0.f)));
                    d0p[o] = dx0;
                    d0p[HW + o] = dx1;
                    d0p[2 * HW + o] = dx2;
                }
                if (dgp) dgp[o] = Df * (dlo + dhi);
                const int pos = cnt[w * NB + bin] + __popc(m & ((1u << lane) - 1u));
                rec[2 * pos] = make_float4(G[0], G[1], G[2], X[0]);
                rec[2 * pos + 1] = make_float4(X[1], X[2], fz, __uint_as_float(((unsigned)r << 16) | (unsigned)c));
            }
            __syncwarp();
            if (ok && lane == __ffs(m) - 1) cnt[w * NB + bin] += __popc(m);
            __syncwarp();
            r = r1;
            cx = cx1;
        }
    }
    __syncthreads();

    // ---- phase 2: d_grid, lane pairs over the bin-sorted records (warp w: a contiguous
    // chunk range); lane 2s+e owns record slot s and coefficient half q = 6e .. 6e+5.
    // The register sums persist across sub-tiles; odd sub-tiles walk the range backwards,
    // so a warp starts a sub-tile in (about) the bin it ended the previous one with.
    {
        const int cbeg = (int)(((long long)nchunks * w) / NW);
        const int cend = (int)(((long long)nchunks * (w + 1)) / NW);
        const bool back = kMulti && (sub & 1) != 0;
        if (!kMulti) {  // one sub-tile: the sums start here (not live across phases 0-1)
#pragma unroll
            for (int k = 0; k < 24; k++) acc2[k] = f2(0.f, 0.f);
            cur_bin = -1;
        }
        for (int it = cbeg; it < cend; it++) {
            const int ch = back ? cend - 1 - (it - cbeg) : it;
            const int bin = chunk_bin[ch];
            if (bin != cur_bin) {
                if (cur_bin >= 0) flush2(cur_bin);
                cur_bin = bin;
            }
            const float4 r0 = rec[2 * (ch * kChunk + slot)], r1 = rec[2 * (ch * kChunk + slot) + 1];
            const unsigned rc = __float_as_uint(r1.w);
            const float fx = fxt[rc & 0xffffu], fy = fyt[rc >> 16], fz = r1.z;
            // this lane's half (q = 4 oc + i): e = 0 owns oc 0 (i = 0..3) and q 8, 9; e = 1 owns
            // oc 1 and q 10, 11 -- the same G / Xt pattern in both halves, three selects
            const float Ga = e1 ? r0.y : r0.x;
            const float Gq[6] = {Ga, Ga, Ga, Ga, r0.z, r0.z};
            const float Xq[6] = {r0.w, r1.x, r1.y, 1.f, e1 ? r1.y : r0.w, e1 ? 1.f : r1.x};
            float2 wt2[4];
            {
                const float2 wx2 = f2(1.f - fx, fx);
                const float wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
#pragma unroll
                for (int pl = 0; pl < 2; pl++)
#pragma unroll
                    for (int bb = 0; bb < 2; bb++) {
                        const float wzy = wz[pl] * wy[bb];
                        wt2[pl * 2 + bb] = __fmul2_rn(f2(wzy, wzy), wx2);
                    }
            }
#pragma unroll
            for (int qq = 0; qq < 6; qq++) {
                const float P = Gq[qq] * Xq[qq];
                const float2 P2 = f2(P, P);
#pragma unroll
                for (int k = 0; k < 4; k++) acc2[k * 6 + qq] = __ffma2_rn(wt2[k], P2, acc2[k * 6 + qq]);
            }
        }
    }
        if (!kMulti && cur_bin >= 0) flush2(cur_bin);
    }  // sub-tiles
    if (kMulti && cur_bin >= 0) flush2(cur_bin);
    __syncthreads();
    // ---- block partial: fixed-order sum over warps
    float *part = partials + (long long)blockIdx.x * 4 * D * 12;
    for (int e = threadIdx.x; e < 4 * D * 12; e += kNT) {
        float s = 0.f;
#pragma unroll
        for (int ww = 0; ww < NW; ww++) s += wacc[ww * 4 * D * 12 + e];
        part[e] = s;
    }
}

// dgrid[n,q,z,y,x] = fixed-order sum of the partials of the dual cells whose
// clamped corners are (y, x).  partial layout: [block][corner][z][q].
// grid (ceil(Gw / 21), Gh D, N): thread t = (q = t % 12, x = 21 blockIdx.x + t / 12) of row y,
// plane z, sample n -- the 12 q of a node are adjacent in a partial, so a warp reads a few
// 48-B runs instead of 32 scattered words (the summation order of every node is fixed).
constexpr int kGX = kThreads / 12;  // 21 grid columns per block
__global__ void __launch_bounds__(kThreads)
    bslice_dgrid_gather(BsliceArgs a, int SY, int SX, const float *__restrict__ partials) {
    const int t = threadIdx.x, q = t % 12, x = blockIdx.x * kGX + t / 12;
    if (t >= 12 * kGX || x >= a.Gw) return;
    const int D = a.D, y = blockIdx.y / D, z = blockIdx.y - y * D, n = blockIdx.z;
    const int per = 4 * D * 12, S = SY * SX;
    float s = 0.f;
    for (int jj = y; jj <= y + 1 && jj <= a.Gh; jj++) {
        for (int b = 0; b < 2; b++) {
            if (clampi(jj - 1 + b, 0, a.Gh - 1) != y) continue;
            for (int kk = x; kk <= x + 1 && kk <= a.Gw; kk++) {
                for (int aa = 0; aa < 2; aa++) {
                    if (clampi(kk - 1 + aa, 0, a.Gw - 1) != x) continue;
                    const long long blk0 = (((long long)n * (a.Gh + 1) + jj) * (a.Gw + 1) + kk) * S;
                    const float *p = partials + blk0 * per + ((b * 2 + aa) * D + z) * 12 + q;
                    for (int st = 0; st < S; st++) s += __ldg(p + (long long)st * per);
                }
            }
        }
    }
    a.dgrid[((((long long)n * 12 + q) * D + z) * a.Gh + y) * a.Gw + x] = s;
}

// ----------------------------------------------------------------- generic (any shape)
// fixed-point exponent of sample n: |sum| <= max|G| max(1, max|X|) * (sum over pixels of
// the trilinear weights of a node <= H W) < 2^61 2^-S (non-finite inputs: S = 0)
RS_DEV int bslice_det_scale(const unsigned *mx, int n, long long HW) {
    const float mg = __uint_as_float(__ldcg(mx + 2 * n)), mxv = fmaxf(1.f, __uint_as_float(__ldcg(mx + 2 * n + 1)));
    if (!(mg > 0.f) || !isfinite(mg) || !isfinite(mxv)) return 0;
    const double bound = (double)mg * (double)mxv * (double)HW;
    return 61 - ilogb(bound) - 1;
}

struct Slice8 {
    int xi[2], yi[2], zi[2];
    float wx[2], wy[2], wz[2];
};

RS_DEV Slice8 slice_geom(const BsliceArgs &a, int y, int x, float g) {
    Slice8 s;
    const double cx = bs_cx(x, a.W, a.Gw), cy = bs_cx(y, a.H, a.Gh), cz = bs_cz(g, a.D);
    const Cell ccx = cell_of(cx), ccy = cell_of(cy), ccz = cell_of(cz);
    s.wx[0] = 1.f - ccx.f; s.wx[1] = ccx.f;
    s.wy[0] = 1.f - ccy.f; s.wy[1] = ccy.f;
    s.wz[0] = 1.f - ccz.f; s.wz[1] = ccz.f;
    for (int t = 0; t < 2; t++) {
        s.xi[t] = clampi(ccx.i0 + t, 0, a.Gw - 1);
        s.yi[t] = clampi(ccy.i0 + t, 0, a.Gh - 1);
        s.zi[t] = clampi(ccz.i0 + t, 0, a.D - 1);
    }
    return s;
}

__global__ void __launch_bounds__(kThreads) bslice_fwd_generic(BsliceArgs a) {
    const long long HW = (long long)a.H * a.W;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= (long long)a.N * HW) return;
    const int n = (int)(idx / HW);
    const long long o = idx - (long long)n * HW;
    const int y = (int)(o / a.W), x = (int)(o - (long long)y * a.W);
    const Slice8 s = slice_geom(a, y, x, __ldg(a.guide + idx));
    const long long plane = (long long)a.Gh * a.Gw;
    const float *g = a.grid + (long long)n * 12 * a.D * plane;
    const float *xp = a.x + (long long)n * 3 * HW + o;
    const float X[3] = {__ldg(xp), __ldg(xp + HW), __ldg(xp + 2 * HW)};
    float A[12];
#pragma unroll
    for (int q = 0; q < 12; q++) A[q] = 0.f;
    for (int e = 0; e < 2; e++)
        for (int b = 0; b < 2; b++)
            for (int aa = 0; aa < 2; aa++) {
                const float wt = s.wz[e] * s.wy[b] * s.wx[aa];
                const long long off = ((long long)s.zi[e] * a.Gh + s.yi[b]) * a.Gw + s.xi[aa];
#pragma unroll
                for (int q = 0; q < 12; q++) A[q] = fmaf(wt, __ldg(g + q * a.D * plane + off), A[q]);
            }
    float *yp = a.y + (long long)n * 3 * HW + o;
#pragma unroll
    for (int oc = 0; oc < 3; oc++)
        yp[oc * HW] = fmaf(A[4 * oc], X[0], fmaf(A[4 * oc + 1], X[1], fmaf(A[4 * oc + 2], X[2], A[4 * oc + 3])));
}

// DET (deterministic=1 on shapes without the tiled path): d_grid by the fixed-point
// integer scatter of det.cuh, specialised here (a term is w * G_o * X~_i, 96 per pixel):
// scale 2^S per sample from max|G| and max(1, max|X|) (bslice_absmax) and the bound
// sum over pixels of w <= H * W, 64-bit integer atomics, one conversion pass.
template <bool DET>
__global__ void __launch_bounds__(kThreads)
    bslice_bwd_generic(BsliceArgs a, unsigned long long *__restrict__ acc, const unsigned *__restrict__ mx) {
    const long long HW = (long long)a.H * a.W;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= (long long)a.N * HW) return;
    const int n = (int)(idx / HW);
    const long long o = idx - (long long)n * HW;
    const int y = (int)(o / a.W), x = (int)(o - (long long)y * a.W);
    const Slice8 s = slice_geom(a, y, x, __ldg(a.guide + idx));
    const long long plane = (long long)a.Gh * a.Gw;
    const float *g = a.grid + (long long)n * 12 * a.D * plane;
    const float *xp = a.x + (long long)n * 3 * HW + o;
    const float *gp = a.dy + (long long)n * 3 * HW + o;
    const float Xt[4] = {__ldg(xp), __ldg(xp + HW), __ldg(xp + 2 * HW), 1.f};
    const float G[3] = {__ldg(gp), __ldg(gp + HW), __ldg(gp + 2 * HW)};
    if (a.dx || a.dguide) {
        // low-plane slice and the slice of the plane difference (P3)
        float Alo[12], Adz[12];
#pragma unroll
        for (int q = 0; q < 12; q++) Alo[q] = Adz[q] = 0.f;
        for (int b = 0; b < 2; b++)
            for (int aa = 0; aa < 2; aa++) {
                const float wt = s.wy[b] * s.wx[aa];
                const long long sp = (long long)s.yi[b] * a.Gw + s.xi[aa];
#pragma unroll
                for (int q = 0; q < 12; q++) {
                    const float gl = __ldg(g + (q * a.D + s.zi[0]) * plane + sp);
                    const float gh = __ldg(g + (q * a.D + s.zi[1]) * plane + sp);
                    Alo[q] = fmaf(wt, gl, Alo[q]);
                    Adz[q] = fmaf(wt, gh - gl, Adz[q]);
                }
            }
        float dgd = 0.f, dx[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int oc = 0; oc < 3; oc++)
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int q = 4 * oc + i;
                const float d = Adz[q];
                if (i < 3) dx[i] = fmaf(G[oc], fmaf(s.wz[1], d, Alo[q]), dx[i]);
                dgd = fmaf(G[oc] * Xt[i], d, dgd);
            }
        if (a.dx) {
            float *dxp = a.dx + (long long)n * 3 * HW + o;
            dxp[0] = dx[0];
            dxp[HW] = dx[1];
            dxp[2 * HW] = dx[2];
        }
        if (a.dguide) a.dguide[idx] = (float)a.D * dgd;
    }
    if (a.dgrid) {
        float *dg = a.dgrid + (long long)n * 12 * a.D * plane;
        int S = 0;
        if (DET) S = bslice_det_scale(mx, n, HW);
        for (int e = 0; e < 2; e++)
            for (int b = 0; b < 2; b++)
                for (int aa = 0; aa < 2; aa++) {
                    const float wt = s.wz[e] * s.wy[b] * s.wx[aa];
                    const long long off = ((long long)s.zi[e] * a.Gh + s.yi[b]) * a.Gw + s.xi[aa];
#pragma unroll
                    for (int oc = 0; oc < 3; oc++)
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            const long long gi = (4 * oc + i) * a.D * plane + off;
                            if (DET) {  // exact fp64 product, one rounding to the fixed point
                                const double v = ldexp((double)wt * (double)G[oc] * (double)Xt[i], S);
                                const long long iv = __double2ll_rn(v);
                                if (iv != 0)
                                    atomicAdd(acc + (long long)n * 12 * a.D * plane + gi, (unsigned long long)iv);
                            } else {
                                red_add(dg + gi, wt * G[oc] * Xt[i]);
                            }
                        }
                }
    }
}

// max |G| and max |X| per sample (order-free atomicMax on the bit patterns)
__global__ void __launch_bounds__(kThreads) bslice_absmax(BsliceArgs a, unsigned *mx) {
    const long long HW = (long long)a.H * a.W;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    const bool in = idx < (long long)a.N * HW;
    const int n = in ? (int)(idx / HW) : 0;
    const long long o = in ? idx - (long long)n * HW : 0;
    unsigned mg = 0u, mxx = 0u;
    if (in)
        for (int i = 0; i < 3; i++) {
            mg = max(mg, __float_as_uint(fabsf(__ldg(a.dy + ((long long)n * 3 + i) * HW + o))));
            mxx = max(mxx, __float_as_uint(fabsf(__ldg(a.x + ((long long)n * 3 + i) * HW + o))));
        }
    // a warp may straddle two samples: reduce per sample index
    const unsigned msk = __match_any_sync(0xffffffffu, in ? n : -1);
    const int leader = __ffs(msk) - 1;
    for (int k = 0; k < 32; k++) {  // segmented max over lanes of the same sample
        const unsigned og = __shfl_sync(0xffffffffu, mg, k), ox = __shfl_sync(0xffffffffu, mxx, k);
        if ((msk >> k) & 1u) {
            mg = max(mg, og);
            mxx = max(mxx, ox);
        }
    }
    if (in && (threadIdx.x & 31) == leader) {
        atomicMax(mx + 2 * n, mg);
        atomicMax(mx + 2 * n + 1, mxx);
    }
}

__global__ void __launch_bounds__(kThreads)
    bslice_dgrid_convert(BsliceArgs a, const unsigned long long *__restrict__ acc, const unsigned *__restrict__ mx) {
    const long long per = 12LL * a.D * a.Gh * a.Gw;
    const long long idx = (long long)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= (long long)a.N * per) return;
    const int n = (int)(idx / per);
    const int S = bslice_det_scale(mx, n, (long long)a.H * a.W);
    a.dgrid[idx] = (float)ldexp((double)(long long)acc[idx], -S);
}

// ----------------------------------------------------------------- d_grid as a pure gather
// GATHER: every grid node (n, y, x) collects its d_grid values by walking all the pixels
// whose clamped corners include it -- the pixels of the dual cells (y-1 .. y) x (x-1 .. x),
// rows [dual_begin(y-1), dual_begin(y+1)) -- and adding w_node * w_z * G_o * X~_i to its
// (q, z) entries: the converted gather of PAPER.md:700-731 in its plain form, with no
// per-dual-cell partials (the comparator of the AUTO dual-cell accumulation, row a11).
// Each pixel is visited by up to 4 nodes.  Per-thread accumulators [q][z][thread] in
// shared memory (no atomics), summed over the threads in a fixed order: deterministic.
constexpr int kNGT = 128;   // threads per node block
constexpr int kNGDMax = 16; // z planes supported (shared memory: 12 * D * kNGT floats)

__global__ void __launch_bounds__(kNGT)
    bslice_dgrid_node_gather(BsliceArgs a, const int *__restrict__ tab) {
    extern __shared__ float nacc[];  // [q][z][thread]
    const int D = a.D;
    const int node = blockIdx.x, n = blockIdx.y;
    const int y = node / a.Gw, x = node - y * a.Gw;
    const int r0 = __ldg(tab + y), r1 = __ldg(tab + y + 2);                      // dual rows y-1 .. y
    const int c0 = __ldg(tab + a.Gh + 2 + x), c1 = __ldg(tab + a.Gh + 2 + x + 2);  // dual cols x-1 .. x
    const int RH = r1 - r0, CW = c1 - c0;
    for (int e = threadIdx.x; e < 12 * D * kNGT; e += kNGT) nacc[e] = 0.f;
    __syncthreads();
    const long long HW = (long long)a.H * a.W;
    const float *gd = a.guide + (long long)n * HW;
    const float *xp = a.x + (long long)n * 3 * HW;
    const float *gp = a.dy + (long long)n * 3 * HW;
    float *my = nacc + threadIdx.x;
    for (int p = threadIdx.x; p < RH * CW; p += kNGT) {
        const int py = r0 + p / CW, px = c0 + p % CW;
        const double cx = bs_cx(px, a.W, a.Gw), cy = bs_cx(py, a.H, a.Gh);
        const Cell ccx = cell_of(cx), ccy = cell_of(cy);
        // this node's share of the pixel's spatial taps (both taps when they clamp onto it)
        const float wx = (clampi(ccx.i0, 0, a.Gw - 1) == x ? 1.f - ccx.f : 0.f) +
                         (clampi(ccx.i0 + 1, 0, a.Gw - 1) == x ? ccx.f : 0.f);
        const float wy = (clampi(ccy.i0, 0, a.Gh - 1) == y ? 1.f - ccy.f : 0.f) +
                         (clampi(ccy.i0 + 1, 0, a.Gh - 1) == y ? ccy.f : 0.f);
        const float wxy = wy * wx;
        if (wxy == 0.f) continue;
        const long long o = (long long)py * a.W + px;
        const double cz = bs_cz(__ldg(gd + o), D);
        const Cell ccz = cell_of(cz);
        const int zl = clampi(ccz.i0, 0, D - 1), zh = clampi(ccz.i0 + 1, 0, D - 1);
        const float wl = wxy * (1.f - ccz.f), wh = wxy * ccz.f;
        const float Xt[4] = {__ldg(xp + o), __ldg(xp + HW + o), __ldg(xp + 2 * HW + o), 1.f};
        const float G[3] = {__ldg(gp + o), __ldg(gp + HW + o), __ldg(gp + 2 * HW + o)};
#pragma unroll
        for (int oc = 0; oc < 3; oc++)
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float P = G[oc] * Xt[i];
                float *q = my + (4 * oc + i) * D * kNGT;
                q[zl * kNGT] = fmaf(wl, P, q[zl * kNGT]);
                q[zh * kNGT] = fmaf(wh, P, q[zh * kNGT]);
            }
    }
    __syncthreads();
    // fixed-order sum over the threads: warp w sums (q, z) rows w, w + 4, ...
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long plane = (long long)a.Gh * a.Gw;
    for (int row = w; row < 12 * D; row += kNGT / 32) {
        const float *rp = nacc + row * kNGT;
        float v = rp[lane] + rp[lane + 32] + rp[lane + 64] + rp[lane + 96];
        v = warp_sum(v);
        if (lane == 0) {
            const int q = row / D, z = row - q * D;
            a.dgrid[(((long long)n * 12 + q) * D + z) * plane + node] = v;
        }
    }
}

// ----------------------------------------------------------------- host-side geometry
struct TileGeom {
    int SY, SX;
    long long blocks;
    bool ok;
};

TileGeom tile_geom(int N, int H, int W, int D, int Gh, int Gw) {
    TileGeom g;
    // dual cells must hold >= 8 px per axis for the tiled kernels to pay off
    g.ok = (W >= 8 * Gw) && (H >= 8 * Gh) && D >= 1 && D <= 64;
    const int maxw = (W + Gw - 1) / Gw, maxh = (H + Gh - 1) / Gh;
    g.SX = (maxw + kTileX - 1) / kTileX;
    g.SY = (maxh + kTileY - 1) / kTileY;
    g.blocks = (long long)N * (Gh + 1) * (Gw + 1) * g.SY * g.SX;
    return g;
}

size_t fwd_smem(int D, int ntab = 1) {
    return sizeof(float4) * 2 * (D + 1) * kPlaneStride + sizeof(float) * (kTileXS + kTileYS) +
           sizeof(float4) * kWarps * ntab * kPlaneStride * (D + 1) + 16;
}

size_t bwd_smem(int D) {
    const int NB = D + 1;
    const int max_chunks = (kTileXS * kTileYS) / kChunk + 1 + NB;
    return sizeof(float4) * 2 * (D + 1) * kPlaneStride + sizeof(float) * (kTileXS + kTileYS) +
           sizeof(float) * kWarps * 4 * D * 12 + sizeof(int) * (kWarps * NB + NB + 1) +
           sizeof(int) * max_chunks + sizeof(unsigned) * max_chunks * kChunk + kTileXS * kTileYS +
           sizeof(float) * kTileXS * kTileYS + 16;
}

size_t split_smem(int D, int NW = kWarps) {
    const int cap = NW == 4 ? 34 * 34 : kV2PX;
    const int NB = D + 1, maxch = cap / kChunk + NB + 1;
    return sizeof(float4) * ((size_t)maxch * kChunk * 2 + (size_t)NB * kBinS) +
           sizeof(float) * ((size_t)cap + kV2TX + 4 + kV2TY + 4 + (size_t)NW * 4 * D * 12) +
           sizeof(int) * ((size_t)NW * NB + NB + 1 + maxch) + cap + 16;
}

// four-warp blocks for dual cells of at most 32 x 32 px (half the d_grid flushes per pixel,
// four blocks per SM); RSGRAD_BSLICE_NW=8 forces the eight-warp form
int split_warps(int H, int W, int Gh, int Gw) {
    const char *e = getenv("RSGRAD_BSLICE_NW");
    if (e && atoi(e) == 8) return 8;
    return ((W + Gw - 1) / Gw <= 32 && (H + Gh - 1) / Gh <= 32) ? 4 : 8;
}

// Backward kernel choice.  bslice_bwd_split where its tile is a whole dual cell (cells of
// <= kV2TX x kV2TY px, two blocks per SM: D <= 9) -- measured 238.6 vs 267.3 us at
// 4 x 1024^2 / 32x32x8 and 855 vs 970 us at 4 x 2048^2 / 64x64x8; for larger cells
// (split into sub-tiles, more d_grid flushes per pixel) bslice_bwd_tiled: 2.52 vs 2.59 ms
// at 64 x 1024^2 / 16x16x8, 193.5 vs 191.5 us at 4 x 1024^2.  RSGRAD_BSLICE_BWD=split|tiled
// forces one (A/B measurements and tests; read per call).
bool use_split(int H, int W, int D, int Gh, int Gw) {
    if (split_smem(D) > (RS_V2MINB >= 2 ? 113 : 226) * 1024) return false;
    const char *e = getenv("RSGRAD_BSLICE_BWD");
    if (e && strcmp(e, "tiled") == 0) return false;
    if (e && strcmp(e, "split") == 0) return true;
    const int maxw = (W + Gw - 1) / Gw, maxh = (H + Gh - 1) / Gh;
    return maxw <= kV2TX && maxh <= 2 * kV2TY;
}

TileGeom tile_geom_split(int N, int H, int W, int D, int Gh, int Gw) {
    TileGeom g = tile_geom(N, H, W, D, Gh, Gw);
    const int maxw = (W + Gw - 1) / Gw, maxh = (H + Gh - 1) / Gh;
    g.SX = (maxw + kV2TX - 1) / kV2TX;
    g.SY = 1;  // (the kernel walks a cell's rows in sub-tiles of <= kV2TY)
    (void)maxh;
    g.blocks = (long long)N * (Gh + 1) * (Gw + 1) * g.SY * g.SX;
    return g;
}

TileGeom bwd_geom(int N, int H, int W, int D, int Gh, int Gw) {
    return use_split(H, W, D, Gh, Gw) ? tile_geom_split(N, H, W, D, Gh, Gw) : tile_geom(N, H, W, D, Gh, Gw);
}

// The tiled backward needs bwd_smem(D) bytes of dynamic shared memory (2056 D + 80740:
// 212 KB at D = 64); it is used only where the current device's opt-in limit allows.
bool bwd_smem_fits(int D) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
        cudaGetLastError();
        optin = 227 * 1024;  // sm_100
    }
    return bwd_smem(D) <= (size_t)optin;
}

}  // namespace

size_t bslice_det_ws_bytes(int N, int D, int Gh, int Gw) {
    return sizeof(unsigned long long) * (size_t)N * 12 * D * Gh * Gw + sizeof(unsigned) * 2 * (size_t)N + 256;
}

size_t bslice_ws_bytes(int N, int H, int W, int D, int Gh, int Gw);
// the workspace a backward call uses: the tiled path's partials, else (deterministic=1)
// the fixed-point d_grid accumulators
size_t bslice_bwd_ws_bytes(int N, int H, int W, int D, int Gh, int Gw, bool det) {
    const size_t t = bslice_ws_bytes(N, H, W, D, Gh, Gw);
    const size_t g = sizeof(int) * (size_t)(Gh + Gw + 4);  // GATHER: the bounds table
    const size_t r = t ? t : (det ? bslice_det_ws_bytes(N, D, Gh, Gw) : 0);
    return r > g ? r : g;
}

size_t bslice_ws_bytes(int N, int H, int W, int D, int Gh, int Gw) {
    const TileGeom g = bwd_geom(N, H, W, D, Gh, Gw);
    if (!g.ok || !bwd_smem_fits(D)) return 0;
    return sizeof(float) * (size_t)g.blocks * 4 * D * 12 + sizeof(int) * (size_t)(Gh + Gw + 4);
}

cudaError_t bslice_fwd_launch(const BsliceArgs &a, cudaStream_t s) {
    const TileGeom g = tile_geom(a.N, a.H, a.W, a.D, a.Gh, a.Gw);
    if (g.ok) {
        // a second row table per warp (narrow dual cells take two rows per item) where it
        // costs little shared memory (D <= ~25)
        const int ntab = fwd_smem(a.D, 2) <= 100 * 1024 ? 2 : 1;
        const size_t sm = fwd_smem(a.D, ntab);
        if (sm > 48 * 1024) {
            cudaError_t ea = cudaFuncSetAttribute(bslice_fwd_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (ea != cudaSuccess) return ea;
        }
        bslice_fwd_tiled<<<(unsigned)g.blocks, kThreads, sm, s>>>(a, g.SY, g.SX, ntab);
    } else {
        const long long total = (long long)a.N * a.H * a.W;
        bslice_fwd_generic<<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
    }
    note_launch();
    return cudaGetLastError();
}

cudaError_t bslice_bwd_launch(const BsliceArgs &a, int algo, int deterministic, void *ws,
                              size_t ws_bytes, cudaStream_t s) {
    const TileGeom g = bwd_geom(a.N, a.H, a.W, a.D, a.Gh, a.Gw);
    const bool split = use_split(a.H, a.W, a.D, a.Gh, a.Gw);
    const bool tiled = g.ok && bwd_smem_fits(a.D) && algo != 3 /*SCATTER_ATOMIC*/ && (algo != 1 /*GATHER*/ || a.D > kNGDMax) && a.dgrid &&
                       ws_bytes >= bslice_ws_bytes(a.N, a.H, a.W, a.D, a.Gh, a.Gw);
    if (tiled) {
        const size_t sm = split ? split_smem(a.D) : bwd_smem(a.D);
        // per device and per call (the attribute belongs to the current device's context)
        const bool multi = split && (a.H + a.Gh - 1) / a.Gh > kV2TY;  // cells of several sub-tiles
        const int nw = split && !multi ? split_warps(a.H, a.W, a.Gh, a.Gw) : 8;
        const size_t smw = split ? split_smem(a.D, nw) : sm;
        cudaError_t ea = cudaFuncSetAttribute(!split ? bslice_bwd_tiled : multi ? bslice_bwd_split<true>
                                                                          : nw == 4 ? bslice_bwd_split<false, 4>
                                                                                    : bslice_bwd_split<false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
        if (ea != cudaSuccess) return ea;
        float *partials = (float *)ws;
        int *tab = (int *)(partials + (size_t)g.blocks * 4 * a.D * 12);
        const int nt = (a.Gh > a.Gw ? a.Gh : a.Gw) + 2;
        // few blocks: the split kernel's blocks search their cell bounds themselves (one launch
        // less: configs[3] 189.4 -> 185.3 us); many small cells: the bounds table (the fp64
        // searches per block cost more: 32x32x8 238.6 vs 246.8 us)
        const bool self_bounds = split && g.blocks <= 2048;
        if (!self_bounds) {
            bslice_bounds_kernel<<<(nt + 127) / 128, 128, 0, s>>>(tab, a.H, a.W, a.Gh, a.Gw);
            note_launch();
        }
        int *stab = self_bounds ? nullptr : tab;
        if (split && multi) bslice_bwd_split<true><<<(unsigned)g.blocks, kThreads, smw, s>>>(a, g.SY, g.SX, partials, stab);
        else if (split && nw == 4)
            bslice_bwd_split<false, 4><<<(unsigned)g.blocks, 128, smw, s>>>(a, g.SY, g.SX, partials, stab);
        else if (split) bslice_bwd_split<false><<<(unsigned)g.blocks, kThreads, smw, s>>>(a, g.SY, g.SX, partials, stab);
        else bslice_bwd_tiled<<<(unsigned)g.blocks, kThreads, sm, s>>>(a, g.SY, g.SX, partials, tab);
        note_launch();
        bslice_dgrid_gather<<<dim3((unsigned)((a.Gw + kGX - 1) / kGX), a.Gh * a.D, a.N), kThreads, 0, s>>>(
            a, g.SY, g.SX, partials);
        note_launch();
    } else if (algo == 1 /*GATHER*/ && a.dgrid && a.D <= kNGDMax) {
        // the pure node gather for d_grid; d_input / d_guide from the per-pixel kernel
        int *tab = (int *)ws;
        const int nt = (a.Gh > a.Gw ? a.Gh : a.Gw) + 2;
        bslice_bounds_kernel<<<(nt + 127) / 128, 128, 0, s>>>(tab, a.H, a.W, a.Gh, a.Gw);
        note_launch();
        if (a.dx || a.dguide) {
            BsliceArgs b = a;
            b.dgrid = nullptr;
            const long long total = (long long)a.N * a.H * a.W;
            bslice_bwd_generic<false><<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(b, nullptr,
                                                                                                           nullptr);
            note_launch();
        }
        const size_t sm = sizeof(float) * 12 * a.D * kNGT;
        cudaError_t ea = cudaFuncSetAttribute(bslice_dgrid_node_gather, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sm);
        if (ea != cudaSuccess) return ea;
        bslice_dgrid_node_gather<<<dim3(a.Gh * a.Gw, a.N), kNGT, sm, s>>>(a, tab);
        note_launch();
    } else if (deterministic && a.dgrid) {
        // deterministic=1 where the tiled path does not apply: fixed-point d_grid
        const long long per = 12LL * a.D * a.Gh * a.Gw;
        unsigned long long *acc = (unsigned long long *)ws;
        unsigned *mx = (unsigned *)(acc + (size_t)a.N * per);
        cudaError_t e = cudaMemsetAsync(ws, 0, bslice_det_ws_bytes(a.N, a.D, a.Gh, a.Gw), s);
        if (e != cudaSuccess) return e;
        const long long total = (long long)a.N * a.H * a.W;
        const unsigned nb = (unsigned)((total + kThreads - 1) / kThreads);
        bslice_absmax<<<nb, kThreads, 0, s>>>(a, mx);
        note_launch();
        bslice_bwd_generic<true><<<nb, kThreads, 0, s>>>(a, acc, mx);
        note_launch();
        bslice_dgrid_convert<<<(unsigned)((a.N * per + kThreads - 1) / kThreads), kThreads, 0, s>>>(a, acc, mx);
        note_launch();
    } else {
        if (a.dgrid) {
            cudaError_t e = cudaMemsetAsync(
                a.dgrid, 0, sizeof(float) * (size_t)a.N * 12 * a.D * a.Gh * a.Gw, s);
            if (e != cudaSuccess) return e;
        }
        const long long total = (long long)a.N * a.H * a.W;
        bslice_bwd_generic<false><<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(a, nullptr,
                                                                                                       nullptr);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace rs
