// stn.cu — spatial transformer (affine_grid + bilinear grid_sample), forward and
// adjoint, sm_100a.  PAPER.md:21-28 (layer), PAPER.md:700-733 (scatter-to-gather
// conversion vs atomics), PAPER.md:838-840 (reductions: partial + serial).
//
// Forward / d_theta (output tiles, stn_out_tile):
//   A block owns a 32x16 tile of OUTPUT pixels.  It computes every pixel's exact
//   fp64 sample coordinate, derives the exact set of input taps the tile reads
//   (per input row: [min x, max x] via shared-memory integer atomics), stages those
//   row segments — the tile's footprint, a parallelogram, ~1.1x the useful bytes —
//   into shared memory with cp.async, CH channels per stage, double-buffered, and
//   gathers the bilinear taps from shared memory.  Global loads are coalesced row
//   segments; the sampling grid is never materialised.
//
// Backward (input tiles, stn_bwd_cell):  "owner computes per floor cell".
//   An output pixel q with floor cell (x0, y0) feeds exactly the four input pixels
//   (x0..x0+1, y0..y0+1).  A block owns a 31x32 tile of input pixels; lane k of
//   warp w owns floor-cell column x0 = xa0-1+k and walks the warp's 4 cell rows.
//   The block stages dY over the exact preimage of its cells (compact rows, per
//   output row i a j-interval from the inverse affine map) plus one 8-byte record
//   per staged output pixel (its exact floor cell and fractions).  For its cell,
//   a lane finds the (~1/det) output pixels whose floor cell it is, reads each dY
//   ONCE per channel and distributes w*dY to its four input pixels in registers;
//   the right neighbour's share arrives by one shuffle and the lower row's share
//   is carried to the next cell row (or across warps through shared memory).
//   This is the scatter-to-gather conversion of PAPER.md:700-731 applied at cell
//   granularity: deterministic, no atomics, no memset.  d_theta is accumulated in
//   the same pass for the cells the tile owns: d_ix = sum_c dY (1-fy)(V01-V00) +
//   fy(V11-V10) from coalesced X loads, times [xt, yt, 1] — warp -> block in fp32,
//   fp64 per-block partials, fixed-order finalize (rfactor).
//
// Fallbacks (decided on the device per sample, no host sync): a sample whose
// affine map is singular or whose preimage exceeds the staging budget takes
// d_theta from stn_out_tile (MODE_DTHETA) and d_input from the atomic scatter
// (PAPER.md:733); border padding (no bounded inverse) always does.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "det.cuh"

namespace rs {
namespace {

constexpr int kThreads = 256;

// RS_RACECHECK_SYNC=1 (a sanitizer build only): every mbarrier hand-off of the stage
// rings is ALSO expressed as cp.async.wait_all + bar.sync, which compute-sanitizer's
// racecheck models (it does not model mbarrier phases); a clean racecheck of that build
// shows the rings have no hazard other than the ones the mbarriers order.
#ifndef RS_RACECHECK_SYNC
#define RS_RACECHECK_SYNC 0
#endif

// forward tiles
constexpr int kFJ = 32;                   // output tile width (px)
#ifndef RS_FIFWD
#define RS_FIFWD 32
#endif
constexpr int kFIfwd = RS_FIFWD, kFIdth = 16;  // output tile rows: forward / d_theta (measured)
constexpr int kFRMax = 128;               // max staged input rows
constexpr int kFStage = 6144;             // floats per pipeline stage

// backward tiles
constexpr int kBX = 31;                   // input px per warp row (32 cell columns)
constexpr int kBRows = 4;                 // px rows per warp
constexpr int kBWarps = 8;
constexpr int kBTY = kBRows * kBWarps;    // 32 px rows per block
constexpr int kBRQMax = 160;              // max staged output rows
constexpr int kBFQMax = 2304;             // max staged output px (records)
constexpr int kBStage = 6144;             // floats per pipeline stage
constexpr int kBCH = 4;                   // max channels per stage (registers)
constexpr int kBHits = 6;                 // cached hits per cell (more: re-searched)

constexpr int MODE_FWD = 0, MODE_DTHETA = 1, MODE_DFLOW = 2;

struct Theta {
    double t[6];
};

RS_DEV Theta load_theta(const float *theta, int n) {
    Theta T;
#pragma unroll
    for (int k = 0; k < 6; k++) T.t[k] = (double)__ldg(theta + 6 * n + k);
    return T;
}

// Exact sample coordinate of output (i, j) from its normalised coords (R1, P1).
RS_DEV void stn_coord(const Theta &T, double xt, double yt, int H, int W, int ac, double &ix,
                      double &iy) {
    ix = stn_unnorm(affine3(T.t[0], T.t[1], T.t[2], xt, yt), W, ac);
    iy = stn_unnorm(affine3(T.t[3], T.t[4], T.t[5], xt, yt), H, ac);
}

// Real-arithmetic affine map q = (j, i) -> p = (ix, iy) and its inverse; used only
// to bound footprints (membership is always decided with the exact coordinate).
struct Affine {
    double m00, m01, m10, m11;  // d p / d q
    double i00, i01, i10, i11;  // inverse
    double p0x, p0y;            // p at q = 0
    double det;
    bool inv;
};

RS_DEV Affine stn_affine(const Theta &T, int H, int W, int Ho, int Wo, int ac) {
    const double ax = ac ? 2.0 / (Wo - 1) : 2.0 / Wo, bx = ac ? -1.0 : 1.0 / Wo - 1.0;
    const double ay = ac ? 2.0 / (Ho - 1) : 2.0 / Ho, by = ac ? -1.0 : 1.0 / Ho - 1.0;
    const double sx = ac ? 0.5 * (W - 1) : 0.5 * W, ox = ac ? 0.0 : -0.5;
    const double sy = ac ? 0.5 * (H - 1) : 0.5 * H, oy = ac ? 0.0 : -0.5;
    Affine A;
    A.m00 = sx * T.t[0] * ax;
    A.m01 = sx * T.t[1] * ay;
    A.m10 = sy * T.t[3] * ax;
    A.m11 = sy * T.t[4] * ay;
    A.p0x = sx * (T.t[0] * bx + T.t[1] * by + T.t[2] + 1.0) + ox;
    A.p0y = sy * (T.t[3] * bx + T.t[4] * by + T.t[5] + 1.0) + oy;
    A.det = A.m00 * A.m11 - A.m01 * A.m10;
    const double scale = fabs(A.m00 * A.m11) + fabs(A.m01 * A.m10);
    A.inv = isfinite(A.det) && fabs(A.det) > 1e-9 * (scale > 0 ? scale : 1.0) && fabs(A.det) > 1e-12;
    const double id = A.inv ? 1.0 / A.det : 0.0;
    A.i00 = A.m11 * id;
    A.i01 = -A.m01 * id;
    A.i10 = -A.m10 * id;
    A.i11 = A.m00 * id;
    return A;
}

// Can the sample take the cell-owner gather (zeros padding only)?  Bounds the
// staged preimage of a block's 32 x 33 cells: rows and records must fit.
RS_DEV bool stn_gatherable(const Affine &A, int Ho, int Wo) {
    if (!A.inv || Ho > 65535 || Wo > 65535) return false;
    const double hq = fabs(A.i10) * (kBX + 1) + fabs(A.i11) * (kBTY + 1);
    const double rq = ceil(hq) + 3.0;
    const double fq = (double)(kBX + 1) * (kBTY + 1) / fabs(A.det) + 8.0 * rq + 64.0;
    // the per-cell candidate window stays small (hits are cached per cell)
    const double wj = fabs(A.i00) + fabs(A.i01), wi = fabs(A.i10) + fabs(A.i11);
    return rq <= kBRQMax && fq <= kBFQMax && (wj + 2.0) * (wi + 2.0) <= 16.0;
}

// ----------------------------------------------------------------- output-tile kernel
// MODE_FWD: y.  MODE_DTHETA: per-tile fp64 partials of d_theta (6 per tile).
// fb_list (optional): loop over the listed samples instead of blockIdx.y.
// FAST (x rows 16-B aligned, affine, no fb_list): 16-B cp.async row copies completing on
// per-stage mbarriers, a compile-time channel-slice stride (immediate smem offsets) with a zero
// slot per slice so every tap is an unpredicated shared load, and for d_theta four
// per-tap accumulators sum_c dY*V (4 FMAs per channel) combined once at the end; with
// ctr (FAST d_theta of every sample) the last tile block of a sample also sums the
// sample's tile partials in tile order into d_theta (no separate finalize launch).
// stage ring: 2 stages of 7168 floats (measured vs 3 x 5120: forward 0.590 vs 0.596 ms,
// backward 1.744 vs 1.774 ms at 16 x 16 x 1024^2; 2 x 9216 drops to 2 blocks per SM)
// d_theta finalize in the last FAST tile block of each sample (1) or a separate launch (0:
// measured 6.96 vs 7.04 ms at 64 x 16 x 1024^2, equal at configs[1]: the per-block fence)
#ifndef RS_DTH_LASTBLOCK
#define RS_DTH_LASTBLOCK 0
#endif
#ifndef RS_NS
#define RS_NS 2
#endif
#ifndef RS_FST
#define RS_FST 7168
#endif
#ifndef RS_FIDF
#define RS_FIDF 32
#endif
#ifndef RS_OT
#define RS_OT 256
#endif
#ifndef RS_OTB
#define RS_OTB 3
#endif
constexpr int kOTFast = RS_OT;     // FAST: threads per output-tile block
constexpr int kOTFastMinB = RS_OTB;
constexpr int kNS = RS_NS;     // FAST: stages in the ring
constexpr int kFSt = RS_FST;   // FAST: floats per stage
constexpr int kFIdf = RS_FIDF; // FAST: d_theta tile rows
static_assert(kFIdf >= 16, "d_theta partials are sized for >= 16-row tiles");
template <int MODE>
struct FastSlices;
template <>
struct FastSlices<0> {  // forward: no dY in the stage
    static constexpr int n = 6;  // channels per stage: 8, 5, 4, 3, 2, 1
    __host__ __device__ static constexpr int cls(int nc) { return (kFSt / nc) & ~3; }
    __host__ __device__ static constexpr int at(int i) {
        return cls(i == 0 ? 8 : 6 - i);
    }
};
template <>
struct FastSlices<1> {  // d_theta: + kFIdf x kFJ dY floats per channel; 5..1 channels per stage
    static constexpr int n = 5;
    __host__ __device__ static constexpr int cls(int nc) { return (kFSt / nc - kFIdf * kFJ) & ~3; }
    __host__ __device__ static constexpr int at(int i) { return cls(5 - i); }
};

// smallest slice stride >= need (the caller guarantees need <= the largest)
template <int I, class FS, class Fn>
RS_DEV void dispatch_slice(int need, Fn &&fn) {
    if constexpr (I == FS::n - 1) {
        fn(std::integral_constant<int, FS::at(I)>{});
    } else {
        if (need <= FS::at(I)) fn(std::integral_constant<int, FS::at(I)>{});
        else dispatch_slice<I + 1, FS>(need, fn);
    }
}

// PRIV (MODE_DTHETA / MODE_DFLOW): d_input by shared-memory privatised scatter: the
// taps add into a footprint-shaped accumulator laid out like the staged X footprint
// (same row table), flushed once per channel chunk with one red.global.add per
// touched footprint element (PAPER.md:733's atomics, made block-local first).
template <int MODE, bool VEC, bool FLOW = false, int kFI = (MODE == 0 ? kFIfwd : kFIdth), bool FAST = false,
          bool PRIV = false>
__global__ void __launch_bounds__(FAST ? kOTFast : kThreads, FAST ? kOTFastMinB : 3)
    stn_out_tile(StnArgs a, const double *__restrict__ xtab, const double *__restrict__ ytab,
                 const int *__restrict__ fb_list, const int *__restrict__ fb_count,
                 double *__restrict__ partials, int tiles_j, int tiles_i, int *__restrict__ ctr = nullptr) {
    constexpr int kOT = FAST ? kOTFast : kThreads, kOW = kOT / 32;  // threads, warps
    constexpr int kFP = kFI / kOW;  // output pixels per thread
    static_assert(kFI % kOW == 0, "every tile row needs a warp: tile rows must be a multiple of the warps");
    extern __shared__ __align__(16) float4 sm4[];
    int *rlo = (int *)sm4;
    int *rhi = rlo + kFRMax;
    int *rxa = rhi + kFRMax;
    int *roff = rxa + kFRMax;
    int *rcnt = roff + kFRMax;
    int *ctl = rcnt + kFRMax;                // 16 ints
    float *stage = (float *)(ctl + 16);      // 2 * kFStage (16-B aligned: 656 ints)
    __shared__ float red[kOT / 32][6];

    __shared__ double ntab[kFJ + kFI];  // normalised coordinates of the tile's columns / rows
    // FAST (single tile per block, fb_list == nullptr): full[s] = TMA bytes landed,
    // empty[s] = all 8 warps done reading stage s
    __shared__ unsigned long long full[kNS], empty[kNS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (FAST && threadIdx.x == 0) {
        for (int b = 0; b < kNS; b++) {
            mbar_init(&full[b], kOT);
            mbar_init(&empty[b], kOT / 32);
        }
        fence_mbar_init();
    }
    const int tj = blockIdx.x % tiles_j, ti = blockIdx.x / tiles_j;
    const long long HW = (long long)a.H * a.W, P = (long long)a.Ho * a.Wo;
    if (!FLOW && threadIdx.x < kFJ + kFI) {
        const bool col = threadIdx.x < kFJ;
        const int idx = col ? tj * kFJ + threadIdx.x : ti * kFI + threadIdx.x - kFJ;
        const int L = col ? a.Wo : a.Ho;
        ntab[threadIdx.x] = idx < L ? ((MODE == MODE_DTHETA && xtab) ? (col ? xtab[idx] : ytab[idx]) : stn_norm(idx, L, a.ac)) : 0.0;
    }
    __syncthreads();
    const int nloop = fb_list ? *fb_count : 1;
    for (int f = 0; f < nloop; f++) {
        const int n = fb_list ? fb_list[f] : blockIdx.y;
        Theta T;
        if (!FLOW) T = load_theta(a.theta, n);
        int x0[kFP], y0[kFP];
        float fx[kFP], fy[kFP], cgx[kFP], cgy[kFP], xtf[kFP], ytf[kFP];
        bool in[kFP], xv0[kFP], xv1[kFP], yv0[kFP], yv1[kFP];
        int ymin = INT_MAX, ymax = INT_MIN;
#pragma unroll
        for (int k = 0; k < kFP; k++) {
            const int i = ti * kFI + warp + kOW * k, j = tj * kFJ + lane;
            in[k] = i < a.Ho && j < a.Wo;
            x0[k] = y0[k] = 0;
            fx[k] = fy[k] = 0.f;
            cgx[k] = cgy[k] = 1.f;
            xtf[k] = ytf[k] = 0.f;
            xv0[k] = xv1[k] = yv0[k] = yv1[k] = false;
            if (in[k]) {
                double ix, iy;
                if (FLOW) {  // FlowNet warp (R4): x + u, y + v in pixels, exact in fp64
                    const float *fp = a.flow + (long long)n * 2 * P + (long long)i * a.Wo + j;
                    ix = __dadd_rn((double)j, (double)ldg_stream(fp));
                    iy = __dadd_rn((double)i, (double)ldg_stream(fp + P));
                } else {
                    const double xt = ntab[lane], yt = ntab[kFJ + warp + kOW * k];
                    xtf[k] = (float)xt;
                    ytf[k] = (float)yt;
                    stn_coord(T, xt, yt, a.H, a.W, a.ac, ix, iy);
                }
                if (a.border) {
                    ix = clamp_coord(ix, a.W, cgx[k]);
                    iy = clamp_coord(iy, a.H, cgy[k]);
                }
                const Cell cx = cell_of(ix), cy = cell_of(iy);
                x0[k] = cx.i0;
                y0[k] = cy.i0;
                fx[k] = cx.f;
                fy[k] = cy.f;
                xv0[k] = cx.i0 >= 0 && cx.i0 < a.W;
                xv1[k] = cx.i0 + 1 >= 0 && cx.i0 + 1 < a.W;
                yv0[k] = cy.i0 >= 0 && cy.i0 < a.H;
                yv1[k] = cy.i0 + 1 >= 0 && cy.i0 + 1 < a.H;
                if (xv0[k] || xv1[k]) {
                    if (yv0[k]) { ymin = min(ymin, y0[k]); ymax = max(ymax, y0[k]); }
                    if (yv1[k]) { ymin = min(ymin, y0[k] + 1); ymax = max(ymax, y0[k] + 1); }
                }
            }
        }
        if (threadIdx.x == 0) {
            ctl[0] = INT_MAX;
            ctl[1] = INT_MIN;
        }
        for (int r = threadIdx.x; r < kFRMax; r += kOT) {
            rlo[r] = INT_MAX;
            rhi[r] = INT_MIN;
        }
        __syncthreads();
        ymin = __reduce_min_sync(0xffffffffu, ymin);
        ymax = __reduce_max_sync(0xffffffffu, ymax);
        if (lane == 0) {
            atomicMin(&ctl[0], ymin);
            atomicMax(&ctl[1], ymax);
        }
        __syncthreads();
        const int ylo = ctl[0];
        const int R = ctl[1] >= ylo ? ctl[1] - ylo + 1 : 0;
        bool fallback = R > kFRMax;
        if (!fallback) {
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                if (!(in[k] && (xv0[k] || xv1[k]))) continue;
                const int xl = xv0[k] ? x0[k] : x0[k] + 1, xh = xv1[k] ? x0[k] + 1 : x0[k];
                if (yv0[k]) { atomicMin(&rlo[y0[k] - ylo], xl); atomicMax(&rhi[y0[k] - ylo], xh); }
                if (yv1[k]) { atomicMin(&rlo[y0[k] + 1 - ylo], xl); atomicMax(&rhi[y0[k] + 1 - ylo], xh); }
            }
        }
        __syncthreads();
        if (!fallback) build_rows<VEC>(R, a.W, rlo, rhi, rxa, roff, rcnt, &ctl[2]);
        __syncthreads();
        if (FAST && !fallback) sum_rows(R, rcnt, &ctl[3]);
        const int F = fallback ? 0 : ctl[2];
        if (FAST) {
            fallback = fallback || F + 4 > FastSlices<MODE == MODE_FWD ? 0 : 1>::at(FastSlices<MODE == MODE_FWD ? 0 : 1>::n - 1);
        } else {
            fallback = fallback || F + ((MODE != MODE_FWD) ? kFI * kFJ : 0) > kFStage;
        }

        float dix[kFP], diy[kFP];
#pragma unroll
        for (int k = 0; k < kFP; k++) dix[k] = diy[k] = 0.f;
        const float *xbase = a.x + (long long)n * a.C * HW;
        if (fallback) {
            // direct global gathers (rare: strongly zoomed-out tiles)
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                if (!in[k]) continue;
                const int i = ti * kFI + warp + kOW * k, j = tj * kFJ + lane;
                const long long o00 = (long long)y0[k] * a.W + x0[k];
                const float w00 = (1.f - fy[k]) * (1.f - fx[k]), w01 = (1.f - fy[k]) * fx[k];
                const float w10 = fy[k] * (1.f - fx[k]), w11 = fy[k] * fx[k];
                for (int c = 0; c < a.C; c++) {
                    const float *p = xbase + (long long)c * HW + o00;
                    const float v00 = (yv0[k] && xv0[k]) ? __ldg(p) : 0.f;
                    const float v01 = (yv0[k] && xv1[k]) ? __ldg(p + 1) : 0.f;
                    const float v10 = (yv1[k] && xv0[k]) ? __ldg(p + a.W) : 0.f;
                    const float v11 = (yv1[k] && xv1[k]) ? __ldg(p + a.W + 1) : 0.f;
                    const long long oo = ((long long)n * a.C + c) * P + (long long)i * a.Wo + j;
                    if (MODE == MODE_FWD) {
                        a.y[oo] = fmaf(w00, v00, fmaf(w01, v01, fmaf(w10, v10, w11 * v11)));
                    } else {
                        const float g = ldg_stream(a.dy + oo);
                        dix[k] = fmaf(g, fmaf(1.f - fy[k], v01 - v00, fy[k] * (v11 - v10)), dix[k]);
                        diy[k] = fmaf(g, fmaf(1.f - fx[k], v10 - v00, fx[k] * (v11 - v01)), diy[k]);
                        if ((MODE == MODE_DFLOW || PRIV) && a.dx) {
                            float *q = a.dx + ((long long)n * a.C + c) * HW + o00;
                            if (yv0[k] && xv0[k]) red_add(q, w00 * g);
                            if (yv0[k] && xv1[k]) red_add(q + 1, w01 * g);
                            if (yv1[k] && xv0[k]) red_add(q + a.W, w10 * g);
                            if (yv1[k] && xv1[k]) red_add(q + a.W + 1, w11 * g);
                        }
                    }
                }
            }
        } else if constexpr (FAST) {
            __syncthreads();  // ctl[3] (sum_rows) visible
            const int Fc = ctl[3];  // floats copied per channel
            // tap offsets into a channel slice; a tap outside the image reads the zero slot F
            int t00[kFP], t01[kFP], t10[kFP], t11[kFP];
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                // a row has a table entry only if one of the pixel's taps in it is in the image
                // (ylo / R come from those): other rows' indices are clamped into the tables
                // (their value is never used) so no read leaves them
                const int r0 = min(max(y0[k] - ylo, 0), kFRMax - 1);
                const int r1 = min(max(y0[k] + 1 - ylo, 0), kFRMax - 1);
                const int s0 = (in[k] && yv0[k]) ? roff[r0] + (x0[k] - rxa[r0]) : 0;
                const int s1 = (in[k] && yv1[k]) ? roff[r1] + (x0[k] - rxa[r1]) : 0;
                t00[k] = (in[k] && yv0[k] && xv0[k]) ? s0 : F;
                t01[k] = (in[k] && yv0[k] && xv1[k]) ? s0 + 1 : F;
                t10[k] = (in[k] && yv1[k] && xv0[k]) ? s1 : F;
                t11[k] = (in[k] && yv1[k] && xv1[k]) ? s1 + 1 : F;
            }
            constexpr int GT = (MODE != MODE_FWD) ? kFI * kFJ : 0;
            const int jb = tj * kFJ;
            const int vrows = min(kFI, a.Ho - ti * kFI), vcols = min(kFJ, a.Wo - jb);
            const int Gc = (MODE != MODE_FWD) ? vrows * vcols : 0;  // dY floats copied per channel
            float acc[kFP][4];
#pragma unroll
            for (int k = 0; k < kFP; k++) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.f;
            auto run = [&](auto ksc) {
                constexpr int kS = decltype(ksc)::value;  // channel slice stride (floats) >= F + 4
                constexpr int NC0 = kFSt / (kS + GT);
                constexpr int NC = NC0 < 8 ? NC0 : 8;
                const int nch = (a.C + NC - 1) / NC;
                for (int e = threadIdx.x; e < kNS * NC * 4; e += kOT)
                    stage[(e / (4 * NC)) * kFSt + ((e >> 2) % NC) * kS + F + (e & 3)] = 0.f;
                __syncthreads();
                const unsigned sstage = smem_u32(stage);
                // every thread issues its share of chunk kc's 16-B cp.async copies and arrives
                // on full[slot] when they have landed (TMA bulk copies are request-rate bound
                // at these 60-130 B row segments: measured 2.7 TB/s at 64 B, scripts/micro)
                // per-thread copy plan, identical for every chunk: four lanes per footprint
                // row (rows tid/4 and tid/4 + 64), eight lanes per dY tile row
                const int q0 = (threadIdx.x & 3) * 4;
                int xnp[2];
                long long xsrc[2];
                unsigned xdst[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int r = MODE == MODE_FWD ? R : (threadIdx.x >> 2) + (kOT / 4) * h;
                    xnp[h] = 0;
                    xsrc[h] = 0;
                    xdst[h] = 0;
                    if (r < R) {
                        const int w = rcnt[r];
                        xnp[h] = w > q0 ? (w - q0 + 15) >> 4 : 0;
                        xsrc[h] = (long long)(ylo + r) * a.W + rxa[r] + q0;
                        xdst[h] = (unsigned)(roff[r] + q0) * 4u;
                    }
                }
                const int gr = threadIdx.x >> 3, gq = (threadIdx.x & 7) * 4;
                const bool gok = MODE != MODE_FWD && gr < vrows && gq < vcols;
                const long long gsrc = (long long)(ti * kFI + gr) * a.Wo + jb + gq;
                const unsigned gdst = (unsigned)(NC * kS + gr * kFJ + gq) * 4u;
                static_assert(kFI * 8 <= kOT || MODE == MODE_FWD, "one dY copy per thread and channel");
                auto issue = [&](int kc) {
                    const int slot = kc % kNS, c0s = kc * NC, ncp = min(NC, a.C - c0s);
                    const unsigned dst = sstage + (unsigned)(slot * kFSt) * 4u;
                    const float *xs = xbase + (long long)c0s * HW;
                    if (MODE == MODE_FWD) {  // (measured faster here than the plan below)
                        for (int r = threadIdx.x >> 2; r < R; r += kOT / 4) {
                            const int w = rcnt[r];
                            const float *src = xs + (long long)(ylo + r) * a.W + rxa[r];
                            unsigned d = dst + (unsigned)roff[r] * 4u;
                            for (int c = 0; c < ncp; c++) {
                                for (int q = q0; q < w; q += 16) cp_async16_s(d + q * 4u, src + q);
                                src += HW;
                                d += kS * 4u;
                            }
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            if (xnp[h] == 0) continue;
                            const float *src = xs + xsrc[h];
                            unsigned d = dst + xdst[h];
                            for (int c = 0; c < ncp; c++) {
                                for (int pc = 0; pc < xnp[h]; pc++) cp_async16_s(d + pc * 64u, src + pc * 16);
                                src += HW;
                                d += kS * 4u;
                            }
                        }
                    }
                    if (gok) {
                        const float *gs = a.dy + ((long long)n * a.C + c0s) * P + gsrc;
                        for (int c = 0; c < ncp; c++) cp_async16_s(dst + gdst + (unsigned)(c * GT) * 4u, gs + (long long)c * P);
                    }
                    cp_async_arrive(&full[slot]);
                };
                for (int kc = 0; kc < kNS - 1 && kc < nch; kc++) issue(kc);
                for (int kc = 0; kc < nch; kc++) {
                    const int c0 = kc * NC, kn = kc + kNS - 1;
                    if (kn < nch) {
                        // slot kn % kNS last held chunk kn - kNS: wait until every warp released it
                        if (kn >= kNS) mbar_wait(&empty[kn % kNS], (unsigned)((kn / kNS - 1) & 1));
                        issue(kn);
                    }
                    mbar_wait(&full[kc % kNS], (unsigned)((kc / kNS) & 1));
                    if (RS_RACECHECK_SYNC) {
                        cp_async_wait<0>();
                        __syncthreads();
                    }
                    const float *S = stage + (kc % kNS) * kFSt;
                    const bool fullc = c0 + NC <= a.C;
#pragma unroll
                    for (int k = 0; k < kFP; k++) {
                        const float *p00 = S + t00[k], *p01 = S + t01[k], *p10 = S + t10[k], *p11 = S + t11[k];
                        if (MODE == MODE_FWD) {
                            if (!in[k]) continue;
                            const float w00 = (1.f - fy[k]) * (1.f - fx[k]), w01 = (1.f - fy[k]) * fx[k];
                            const float w10 = fy[k] * (1.f - fx[k]), w11 = fy[k] * fx[k];
                            const int i = ti * kFI + warp + kOW * k, j = jb + lane;
                            float *yp = a.y + ((long long)n * a.C + c0) * P + (long long)i * a.Wo + j;
#pragma unroll
                            for (int c = 0; c < NC; c++) {
                                if (!fullc && c0 + c >= a.C) break;
                                const float v = fmaf(w00, p00[c * kS], fmaf(w01, p01[c * kS],
                                                     fmaf(w10, p10[c * kS], w11 * p11[c * kS])));
                                yp[(long long)c * P] = v;
                            }
                        } else {
                            const float *gp = S + NC * kS + (warp + kOW * k) * kFJ + lane;
#pragma unroll
                            for (int c = 0; c < NC; c++) {
                                if (!fullc && c0 + c >= a.C) break;
                                const float g = gp[c * GT];
                                acc[k][0] = fmaf(g, p00[c * kS], acc[k][0]);
                                acc[k][1] = fmaf(g, p01[c * kS], acc[k][1]);
                                acc[k][2] = fmaf(g, p10[c * kS], acc[k][2]);
                                acc[k][3] = fmaf(g, p11[c * kS], acc[k][3]);
                            }
                        }
                    }
                    __syncwarp();
                    if (RS_RACECHECK_SYNC) __syncthreads();
                    if (lane == 0) mbar_arrive(&empty[kc % kNS]);
                }
            };
            dispatch_slice<0, FastSlices<MODE == MODE_FWD ? 0 : 1>>(F + 4, run);
            if (MODE != MODE_FWD) {
#pragma unroll
                for (int k = 0; k < kFP; k++) {  // d_ix = sum_c dY dV/dx, d_iy likewise (R1)
                    dix[k] = fmaf(1.f - fy[k], acc[k][1] - acc[k][0], fy[k] * (acc[k][3] - acc[k][2]));
                    diy[k] = fmaf(1.f - fx[k], acc[k][2] - acc[k][0], fx[k] * (acc[k][3] - acc[k][1]));
                }
            }
        } else {
            int s0[kFP], s1[kFP];
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                const int r0 = min(max(y0[k] - ylo, 0), kFRMax - 1);  // as above: clamped rows
                const int r1 = min(max(y0[k] + 1 - ylo, 0), kFRMax - 1);
                s0[k] = (in[k] && yv0[k]) ? roff[r0] + (x0[k] - rxa[r0]) : 0;
                s1[k] = (in[k] && yv1[k]) ? roff[r1] + (x0[k] - rxa[r1]) : 0;
            }
            // d_theta also stages the tile's dY rows (kFI x kFJ per channel) after the X footprint
            constexpr int GT = (MODE != MODE_FWD) ? kFI * kFJ : 0;
            const int CH = min(a.C, kFStage / (F + GT > 0 ? F + GT : 1));
            const int nch = (a.C + CH - 1) / CH;
            const bool gvec = (a.Wo % 4 == 0) && (((uintptr_t)a.dy & 15u) == 0);
            auto stage_g = [&](float *dst, int c0s, int ncp) {
                if (MODE == MODE_FWD) return;
                const int jb = tj * kFJ;
                if (gvec) {
                    for (int e = threadIdx.x; e < ncp * kFI * (kFJ / 4); e += kOT) {
                        const int c = e / (kFI * (kFJ / 4)), rem = e - c * (kFI * (kFJ / 4));
                        const int r = rem / (kFJ / 4), q4 = (rem - r * (kFJ / 4)) * 4;
                        const int i = ti * kFI + r;
                        if (i < a.Ho && jb + q4 < a.Wo)
                            cp_async16(dst + c * GT + r * kFJ + q4,
                                       a.dy + ((long long)n * a.C + c0s + c) * P + (long long)i * a.Wo + jb + q4);
                    }
                } else {
                    for (int e = threadIdx.x; e < ncp * kFI * kFJ; e += kOT) {
                        const int c = e / (kFI * kFJ), rem = e - c * (kFI * kFJ);
                        const int r = rem / kFJ, q = rem - r * kFJ;
                        const int i = ti * kFI + r;
                        if (i < a.Ho && jb + q < a.Wo)
                            cp_async4(dst + c * GT + r * kFJ + q,
                                      a.dy + ((long long)n * a.C + c0s + c) * P + (long long)i * a.Wo + jb + q);
                    }
                }
            };
            float *pacc = stage + 2 * kFStage;  // PRIV: CH x F accumulator (CH * F <= kFStage)
            if (PRIV && a.dx)
                for (int e = threadIdx.x; e < CH * F; e += kOT) pacc[e] = 0.f;
            if (F > 0) stage_rows<VEC>(stage, F, xbase, HW, min(CH, a.C), R, a.W, ylo, rxa, roff, rcnt);
            stage_g(stage + CH * F, 0, min(CH, a.C));
            cp_async_commit();
            for (int kc = 0; kc < nch; kc++) {
                const int c0 = kc * CH, cn = min(CH, a.C - c0);
                if (kc + 1 < nch) {
                    float *nxt = stage + ((kc + 1) & 1) * kFStage;
                    if (F > 0)
                        stage_rows<VEC>(nxt, F, xbase + (long long)(c0 + CH) * HW,
                                        HW, min(CH, a.C - c0 - CH), R, a.W, ylo, rxa, roff, rcnt);
                    stage_g(nxt + CH * F, c0 + CH, min(CH, a.C - c0 - CH));
                    cp_async_commit();
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const float *S = stage + (kc & 1) * kFStage;
#pragma unroll
                for (int k = 0; k < kFP; k++) {
                    if (!in[k]) continue;
                    const int i = ti * kFI + warp + kOW * k, j = tj * kFJ + lane;
                    const bool k00 = yv0[k] && xv0[k], k01 = yv0[k] && xv1[k];
                    const bool k10 = yv1[k] && xv0[k], k11 = yv1[k] && xv1[k];
                    const float w00 = (1.f - fy[k]) * (1.f - fx[k]), w01 = (1.f - fy[k]) * fx[k];
                    const float w10 = fy[k] * (1.f - fx[k]), w11 = fy[k] * fx[k];
                    const long long ob = ((long long)n * a.C + c0) * P + (long long)i * a.Wo + j;
#pragma unroll 4
                    for (int c = 0; c < cn; c++) {
                        const float *Sc = S + c * F;
                        const float v00 = k00 ? Sc[s0[k]] : 0.f, v01 = k01 ? Sc[s0[k] + 1] : 0.f;
                        const float v10 = k10 ? Sc[s1[k]] : 0.f, v11 = k11 ? Sc[s1[k] + 1] : 0.f;
                        if (MODE == MODE_FWD) {
                            a.y[ob + c * P] = fmaf(w00, v00, fmaf(w01, v01, fmaf(w10, v10, w11 * v11)));
                        } else {
                            const float g = S[CH * F + c * GT + (warp + kOW * k) * kFJ + lane];
                            dix[k] = fmaf(g, fmaf(1.f - fy[k], v01 - v00, fy[k] * (v11 - v10)), dix[k]);
                            diy[k] = fmaf(g, fmaf(1.f - fx[k], v10 - v00, fx[k] * (v11 - v01)), diy[k]);
                            if (PRIV && a.dx) {  // block-private accumulator (shared atomics)
                                float *pc = pacc + c * F;
                                if (k00) atomicAdd(pc + s0[k], w00 * g);
                                if (k01) atomicAdd(pc + s0[k] + 1, w01 * g);
                                if (k10) atomicAdd(pc + s1[k], w10 * g);
                                if (k11) atomicAdd(pc + s1[k] + 1, w11 * g);
                            } else if (MODE == MODE_DFLOW && a.dx) {  // no bounded inverse: atomic scatter
                                float *q = a.dx + ((long long)n * a.C + c0 + c) * HW +
                                           (long long)y0[k] * a.W + x0[k];
                                if (k00) red_add(q, w00 * g);
                                if (k01) red_add(q + 1, w01 * g);
                                if (k10) red_add(q + a.W, w10 * g);
                                if (k11) red_add(q + a.W + 1, w11 * g);
                            }
                        }
                    }
                }
                __syncthreads();
                if (PRIV && a.dx) {
                    // flush: one red per touched footprint element, then re-zero (8 lanes per row)
                    float *dxc = a.dx + ((long long)n * a.C + c0) * HW;
                    for (int r = (threadIdx.x >> 3); r < R; r += kOT / 8) {
                        const int wdt = rcnt[r];
                        float *gr = dxc + (long long)(ylo + r) * a.W + rxa[r];
                        for (int c = 0; c < cn; c++) {
                            float *pr = pacc + c * F + roff[r];
                            for (int q = threadIdx.x & 7; q < wdt; q += 8) {
                                const float v = pr[q];
                                if (v != 0.f) {
                                    red_add(gr + (long long)c * HW + q, v);
                                    pr[q] = 0.f;
                                }
                            }
                        }
                    }
                    __syncthreads();
                }
            }
        }
        if (MODE == MODE_DFLOW && a.dflow) {
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                if (!in[k]) continue;
                const int i = ti * kFI + warp + kOW * k, j = tj * kFJ + lane;
                float *dfp = a.dflow + (long long)n * 2 * P + (long long)i * a.Wo + j;
                dfp[0] = dix[k] * cgx[k];
                dfp[P] = diy[k] * cgy[k];
            }
        }
        if (MODE == MODE_DTHETA) {
            const float sx = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W;
            const float sy = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
            float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < kFP; k++) {
                if (!in[k]) continue;
                const float dgx = dix[k] * sx * cgx[k], dgy = diy[k] * sy * cgy[k];
                acc[0] = fmaf(dgx, xtf[k], acc[0]);
                acc[1] = fmaf(dgx, ytf[k], acc[1]);
                acc[2] += dgx;
                acc[3] = fmaf(dgy, xtf[k], acc[3]);
                acc[4] = fmaf(dgy, ytf[k], acc[4]);
                acc[5] += dgy;
            }
#pragma unroll
            for (int k = 0; k < 6; k++) {
                const float v = warp_sum(acc[k]);
                if (lane == 0) red[warp][k] = v;
            }
            __syncthreads();
            if (threadIdx.x < 6) {
                double s = 0.0;
                for (int w = 0; w < kOT / 32; w++) s += (double)red[w][threadIdx.x];
                partials[((long long)n * tiles_j * tiles_i + blockIdx.x) * 6 + threadIdx.x] = s;
            }
            if (ctr) {
                // the last tile block of sample n sums its tiles' partials in tile order
                // (the fixed order of stn_dtheta_finalize: bitwise the same result) and
                // writes d_theta -- one launch less per call
                __shared__ int last;
                if (threadIdx.x < 6) __threadfence();  // the partial writers publish
                __syncthreads();
                if (threadIdx.x == 0) last = atomicAdd(ctr + n, 1) == (int)gridDim.x - 1;
                __syncthreads();
                if (last) {
                    __threadfence();
                    const double *pp = partials + (long long)n * tiles_j * tiles_i * 6;
                    const int nt = tiles_j * tiles_i;
                    double sk[6] = {0, 0, 0, 0, 0, 0};
                    for (int b = threadIdx.x; b < nt; b += kOT)
#pragma unroll
                        for (int k = 0; k < 6; k++) sk[k] += __ldcg(pp + (long long)b * 6 + k);
                    __shared__ double redd[kOT / 32][6];
#pragma unroll
                    for (int k = 0; k < 6; k++) {
                        const double v = warp_sum_d(sk[k]);
                        if (lane == 0) redd[warp][k] = v;
                    }
                    __syncthreads();
                    if (threadIdx.x < 6) {
                        double v = 0.0;
                        for (int w = 0; w < kOT / 32; w++) v += redd[w][threadIdx.x];
                        a.dtheta[6 * n + threadIdx.x] = (float)v;
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------- backward: tables + classify

RS_DEV bool stn_gather_ok(const Affine &A, int Ho, int Wo);
RS_DEV bool stn_lean_ok(const Affine &A, int Ho, int Wo);

// flags[n] = 1 if sample n takes the gather adjoint (variant 0: cell-owner,
// 1: per-pixel gather, 2: lean); fb_list = the others.  Called by one whole block.
RS_DEV bool stn_heavy(const Affine &A, int border, int H, int W, int Ho, int Wo);

RS_DEV void stn_classify_block(const StnArgs &a, int allow_gather, int variant, int *flags, int *fb_list,
                               int *fb_count, int *hv_list, int *hv_count, unsigned *det_slots) {
    __shared__ int cnt, hcnt;
    if (threadIdx.x == 0) cnt = hcnt = 0;
    for (int e = threadIdx.x; e < a.N + 2; e += blockDim.x) det_slots[e] = 0u;  // det.cuh bar + max slots
    __syncthreads();
    for (int n = threadIdx.x; n < a.N; n += blockDim.x) {
        const Theta T = load_theta(a.theta, n);
        const Affine A = stn_affine(T, a.H, a.W, a.Ho, a.Wo, a.ac);
        const bool g = allow_gather && !a.border &&
                       (variant == 1 ? stn_gather_ok(A, a.Ho, a.Wo)
                                     : variant == 2 ? stn_lean_ok(A, a.Ho, a.Wo) : stn_gatherable(A, a.Ho, a.Wo));
        flags[n] = g ? 1 : 0;
        if (!g) fb_list[atomicAdd(&cnt, 1)] = n;
        if (!g && stn_heavy(A, a.border, a.H, a.W, a.Ho, a.Wo)) hv_list[atomicAdd(&hcnt, 1)] = n;  // exact scatter (AUTO's atomics skip it)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *fb_count = cnt;
        *hv_count = hcnt;
    }
}

// One launch for the per-call preparation: the normalised coordinate tables (every
// block), the per-sample classification and the d_theta tile counters (block 0).
__global__ void stn_prep_kernel(StnArgs a, int allow_gather, int variant, double *xt, double *yt, int *flags,
                                int *fb_list, int *fb_count, int *ctr, int *hv_list, int *hv_count,
                                unsigned *det_slots) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < a.Wo) xt[t] = stn_norm(t, a.Wo, a.ac);
    if (t < a.Ho) yt[t] = stn_norm(t, a.Ho, a.ac);
    if (blockIdx.x == 0) {
        for (int n = threadIdx.x; n < a.N; n += blockDim.x) ctr[n] = 0;
        stn_classify_block(a, allow_gather, variant, flags, fb_list, fb_count, hv_list, hv_count, det_slots);
    }
}

// ----------------------------------------------------------------- backward: cell-owner gather
RS_DEV uint2 pack_rec(int cx, int cy, float fx, float fy) {
    unsigned ux = (unsigned)(fx * 16777216.0f + 0.5f), uy = (unsigned)(fy * 16777216.0f + 0.5f);
    ux = ux > 0xffffffu ? 0xffffffu : ux;
    uy = uy > 0xffffffu ? 0xffffffu : uy;
    return make_uint2(((unsigned)cx << 24) | ux, ((unsigned)cy << 24) | uy);
}

#ifndef RS_CELL_MINB
#define RS_CELL_MINB 2
#endif
template <bool VEC>
__global__ void __launch_bounds__(kThreads, RS_CELL_MINB)
    stn_bwd_cell(StnArgs a, const double *__restrict__ xtab, const double *__restrict__ ytab,
                 const int *__restrict__ flags, double *__restrict__ partials, int tiles_x,
                 int tiles_y) {
    extern __shared__ __align__(16) float4 sm4[];
    float *stage = (float *)sm4;                               // 2 * kBStage
    uint2 *rec = (uint2 *)(stage + 2 * kBStage);               // kBFQMax
    unsigned *ijs = (unsigned *)(rec + kBFQMax);               // kBFQMax
    int4 *rowt = (int4 *)(ijs + kBFQMax);                      // kBRQMax {lo, hi, off - xa, -}
    int *qlo = (int *)(rowt + kBRQMax);
    int *qhi = qlo + kBRQMax;
    int *qxa = qhi + kBRQMax;
    int *qoff = qxa + kBRQMax;
    int *qcnt = qoff + kBRQMax;
    int *ctl = qcnt + kBRQMax;                                  // 8
    float *carry = (float *)(ctl + 8);                          // kBWarps * 2 * kBCH * 32
    unsigned short *hlist = (unsigned short *)(carry + kBWarps * 2 * kBCH * 32);  // [warp][row][hit][lane]
    unsigned char *hcnt = (unsigned char *)(hlist + kBWarps * (kBRows + 1) * kBHits * 32);  // [warp][row][lane]
    __shared__ float red[kBWarps][6];

    const int n = blockIdx.y;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int xa0 = tx * kBX, yb0 = ty * kBTY;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long HW = (long long)a.H * a.W, P = (long long)a.Ho * a.Wo;
    const int px = xa0 - 1 + lane;  // this lane's cell column == the px column it finalises
    float *dxn = a.dx ? a.dx + (long long)n * a.C * HW : nullptr;
    double *part = partials + ((long long)n * tiles_x * tiles_y + blockIdx.x) * 6;

    if (!flags[n]) {  // fallback sample: zero this tile's dx (atomic scatter adds later)
        if (dxn && lane >= 1 && px < a.W)
            for (int r = warp; r < kBTY; r += kBWarps) {
                const int y = yb0 + r;
                if (y < a.H)
                    for (int c = 0; c < a.C; c++) dxn[(long long)c * HW + (long long)y * a.W + px] = 0.f;
            }
        if (threadIdx.x < 6) part[threadIdx.x] = 0.0;
        return;
    }
    const Theta T = load_theta(a.theta, n);
    const Affine A = stn_affine(T, a.H, a.W, a.Ho, a.Wo, a.ac);

    // ---- preimage rows of the cells [xa0-1, xa0+kBX-1] x [yb0-1, yb0+kBTY-1]
    const double eps = 1e-3;
    const double Lx = xa0 - 1 - eps, Ux = xa0 + kBX + eps;
    const double Ly = yb0 - 1 - eps, Uy = yb0 + kBTY + eps;
    double imin = 1e300, imax = -1e300;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const double px_ = (c & 1) ? Ux : Lx, py_ = (c & 2) ? Uy : Ly;
        const double qi = A.i10 * (px_ - A.p0x) + A.i11 * (py_ - A.p0y);
        imin = fmin(imin, qi);
        imax = fmax(imax, qi);
    }
    const int ilo = max(0, (int)ceil(fmax(imin, -1e9)));
    const int ihi = min(a.Ho - 1, (int)floor(fmin(imax, 1e9)));
    const int RQ = min(kBRQMax, max(0, ihi - ilo + 1));
    for (int r = threadIdx.x; r < RQ; r += kThreads) {
        const int i = ilo + r;
        double jl = -1e300, jh = 1e300;
        // strip constraints  L <= m_0 j + m_1 i + p0 <= U  for x and y
        const double ax_[2] = {A.m00, A.m10}, bx_[2] = {A.m01 * i + A.p0x, A.m11 * i + A.p0y};
        const double L_[2] = {Lx, Ly}, U_[2] = {Ux, Uy};
#pragma unroll
        for (int d = 0; d < 2; d++) {
            if (fabs(ax_[d]) < 1e-12) {
                if (bx_[d] < L_[d] || bx_[d] > U_[d]) { jl = 1e300; jh = -1e300; }
            } else {
                double u = (L_[d] - bx_[d]) / ax_[d], v = (U_[d] - bx_[d]) / ax_[d];
                if (u > v) { const double t = u; u = v; v = t; }
                jl = fmax(jl, u);
                jh = fmin(jh, v);
            }
        }
        const int lo = max(0, (int)ceil(fmax(jl, -1e9))), hi = min(a.Wo - 1, (int)floor(fmin(jh, 1e9)));
        qlo[r] = lo;
        qhi[r] = hi;
    }
    __syncthreads();
    build_rows<VEC>(RQ, a.Wo, qlo, qhi, qxa, qoff, qcnt, &ctl[0]);
    __syncthreads();
    const int FQ = min(ctl[0], kBFQMax);
    for (int r = threadIdx.x; r < RQ; r += kThreads) rowt[r] = make_int4(qlo[r], qhi[r], qoff[r] - qxa[r], 0);
    // ---- records: exact floor cell (relative to the block's cell origin) + fractions
    for (int r = warp; r < RQ; r += kBWarps) {
        const int i = ilo + r;
        const double yt = ytab[i];
        const int wr = (qcnt[r] + 3) & ~3;
        for (int col = lane; col < wr; col += 32) {
            const int j = qxa[r] + col, e = qoff[r] + col;
            if (e >= kBFQMax) break;
            uint2 R = make_uint2(0xff000000u, 0xff000000u);
            if (col < qcnt[r] && j >= qlo[r] && j <= qhi[r]) {
                double ix, iy;
                stn_coord(T, xtab[j], yt, a.H, a.W, a.ac, ix, iy);
                const Cell cx = cell_of(ix), cy = cell_of(iy);
                const int rx = cx.i0 - (xa0 - 1), ry = cy.i0 - (yb0 - 1);
                if (rx >= 0 && rx <= kBX && ry >= 0 && ry <= kBTY) R = pack_rec(rx, ry, cx.f, cy.f);
            }
            rec[e] = R;
            ijs[e] = ((unsigned)i << 16) | (unsigned)j;
        }
    }
    const int CH = min(min(a.C, kBCH), FQ > 0 ? max(1, kBStage / FQ) : kBCH);
    const int nch = (a.C + CH - 1) / CH;
    const float *gbase = a.dy + (long long)n * a.C * P;
    const float *xbase = a.x + (long long)n * a.C * HW;
    __syncthreads();
    if (FQ > 0) stage_rows<VEC>(stage, FQ, gbase, P, min(CH, a.C), RQ, a.Wo, ilo, qxa, qoff, qcnt);
    cp_async_commit();

    // warp geometry: warp 0 also walks the halo cell row yb0-1
    const int wy0 = (warp == 0) ? yb0 - 1 : yb0 + kBRows * warp;
    const int nrows = (warp == 0) ? kBRows + 1 : kBRows;
    const bool ownx = (px >= xa0) || (px == -1);
    const bool pxin = lane >= 1 && px < a.W;
    const bool vx0 = px >= 0 && px < a.W, vx1 = px + 1 < a.W;
    const unsigned cxw = (unsigned)(px - (xa0 - 1));
    const double hj1 = 0.5 * (fabs(A.i00) + fabs(A.i01)) + eps, hi1 = 0.5 * (fabs(A.i10) + fabs(A.i11)) + eps;
    unsigned short *myhl = hlist + warp * (kBRows + 1) * kBHits * 32 + lane;
    unsigned char *myhc = hcnt + warp * (kBRows + 1) * 32 + lane;

    // ---- search (overlaps the first stage's copy): output pixels whose floor cell is (px, y0)
    auto search = [&](int y0, int rr, bool store, auto &&fn) {
        const unsigned cyw = (unsigned)(y0 - (yb0 - 1));
        const double ux = (double)px + 0.5 - A.p0x, uy = (double)y0 + 0.5 - A.p0y;
        const double qj = A.i00 * ux + A.i01 * uy, qi = A.i10 * ux + A.i11 * uy;
        const int jl = (int)ceil(qj - hj1), jh = (int)floor(qj + hj1);
        const int il = max(ilo, (int)ceil(qi - hi1)), ih = min(ilo + RQ - 1, (int)floor(qi + hi1));
        int cnt = 0;
        for (int i = il; i <= ih; i++) {
            const int4 rt = rowt[i - ilo];
            const int ja = max(jl, rt.x), jb = min(jh, rt.y);
            for (int j = ja; j <= jb; j++) {
                const int e = rt.z + j;
                const uint2 R = rec[e];
                if ((R.x >> 24) == cxw && (R.y >> 24) == cyw) {
                    if (store && cnt < kBHits) myhl[(rr * kBHits + cnt) * 32] = (unsigned short)e;
                    fn(e);
                    cnt++;
                }
            }
        }
        if (store) myhc[rr * 32] = (unsigned char)(cnt > kBHits ? 255 : cnt);
    };
    for (int rr = 0; rr < nrows; rr++) search(wy0 + rr, rr, true, [](int) {});

    float acc6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float sxs = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W;
    const float sys = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
    const float axf = a.ac ? 2.f / (a.Wo - 1) : 2.f / a.Wo, bxf = a.ac ? -1.f : 1.f / a.Wo - 1.f;
    const float ayf = a.ac ? 2.f / (a.Ho - 1) : 2.f / a.Ho, byf = a.ac ? -1.f : 1.f / a.Ho - 1.f;


    // One chunk of NC channels (compile-time, so no predicated-off channel work).
    auto run_chunk = [&](const float *S, int c0, auto ncc) {
        constexpr int NC = decltype(ncc)::value;
        const float *xch = xbase + (long long)c0 * HW + px;
        float *dxc = dxn ? dxn + (long long)c0 * HW + px : nullptr;
        float L[NC], Rr[NC], NL[NC], NR[NC], FL[NC], FR[NC], xc0[NC], xc1[NC];
        const bool yv0 = wy0 >= 0 && wy0 < a.H;
#pragma unroll
        for (int c = 0; c < NC; c++) {
            NL[c] = NR[c] = FL[c] = FR[c] = 0.f;
            const float *p = xch + (long long)c * HW + (long long)wy0 * a.W;
            xc0[c] = (yv0 && vx0) ? __ldg(p) : 0.f;
            xc1[c] = (yv0 && vx1) ? __ldg(p + 1) : 0.f;
        }
        const float *xrow = xch + (long long)(wy0 + 1) * a.W;
        float *drow = dxc ? dxc + (long long)wy0 * a.W : nullptr;
#pragma unroll 1
        for (int rr = 0; rr < nrows; rr++, xrow += a.W, drow += a.W) {
            const int y0 = wy0 + rr;
            const bool owned = ownx && ((y0 >= yb0) || (y0 == -1));
            const bool yv = y0 + 1 >= 0 && y0 + 1 < a.H;
            float dxa[NC], ddx[NC], dya[NC], ddy[NC];
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const float *p = xrow + (long long)c * HW;
                const float n0 = (yv && vx0) ? __ldg(p) : 0.f;
                const float n1 = (yv && vx1) ? __ldg(p + 1) : 0.f;
                dxa[c] = xc1[c] - xc0[c];
                ddx[c] = (n1 - n0) - dxa[c];
                dya[c] = n0 - xc0[c];
                ddy[c] = (n1 - xc1[c]) - dya[c];
                xc0[c] = n0;
                xc1[c] = n1;
                L[c] = NL[c];
                Rr[c] = NR[c];
                NL[c] = 0.f;
                NR[c] = 0.f;
            }
            auto process = [&](int e) {
                const uint2 R = rec[e];
                const float fx = (float)(R.x & 0xffffffu) * (1.f / 16777216.f);
                const float fy = (float)(R.y & 0xffffffu) * (1.f / 16777216.f);
                const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
                const float w10 = fy * (1.f - fx), w11 = fy * fx;
                float dq = 0.f, dr = 0.f;
                const float *Se = S + e;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const float g = Se[c * FQ];
                    L[c] = fmaf(w00, g, L[c]);
                    Rr[c] = fmaf(w01, g, Rr[c]);
                    NL[c] = fmaf(w10, g, NL[c]);
                    NR[c] = fmaf(w11, g, NR[c]);
                    dq = fmaf(g, fmaf(fy, ddx[c], dxa[c]), dq);
                    dr = fmaf(g, fmaf(fx, ddy[c], dya[c]), dr);
                }
                if (owned) {
                    const unsigned ij = ijs[e];
                    const float xt = fmaf(axf, (float)(ij & 0xffffu), bxf);
                    const float yt = fmaf(ayf, (float)(ij >> 16), byf);
                    const float dgx = dq * sxs, dgy = dr * sys;
                    acc6[0] = fmaf(dgx, xt, acc6[0]);
                    acc6[1] = fmaf(dgx, yt, acc6[1]);
                    acc6[2] += dgx;
                    acc6[3] = fmaf(dgy, xt, acc6[3]);
                    acc6[4] = fmaf(dgy, yt, acc6[4]);
                    acc6[5] += dgy;
                }
            };
            const int hn = myhc[rr * 32];
            const int hmax = __reduce_max_sync(0xffffffffu, hn == 255 ? 0 : hn);
            if (hn == 255) {
                search(y0, rr, false, process);  // > kBHits output pixels in this cell (rare)
            } else {
                for (int h = 0; h < hmax; h++)
                    if (h < hn) process(myhl[(rr * kBHits + h) * 32]);
            }
            // ---- finalise px row y0: own left share + left neighbour's right share
            if (y0 >= yb0) {
                if (warp > 0 && rr == 0) {  // needs the warp above's carry: after the barrier
#pragma unroll
                    for (int c = 0; c < NC; c++) { FL[c] = L[c]; FR[c] = Rr[c]; }
                } else {
                    const bool wr = drow && pxin && y0 < a.H;
#pragma unroll
                    for (int c = 0; c < NC; c++) {
                        const float v = L[c] + __shfl_up_sync(0xffffffffu, Rr[c], 1);
                        if (wr) drow[(long long)c * HW] = v;
                    }
                }
            }
        }
        // ---- carry the last cell row's lower share to the warp below
        if (warp < kBWarps - 1) {
            float *cw = carry + warp * 2 * kBCH * 32;
#pragma unroll
            for (int c = 0; c < NC; c++) { cw[c * 32 + lane] = NL[c]; cw[(kBCH + c) * 32 + lane] = NR[c]; }
        }
        __syncthreads();
        if (warp > 0) {
            const float *cu = carry + (warp - 1) * 2 * kBCH * 32;
            const int y = yb0 + kBRows * warp;
            const bool wr = dxc && pxin && y < a.H;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const float l = FL[c] + cu[c * 32 + lane], r = FR[c] + cu[(kBCH + c) * 32 + lane];
                const float v = l + __shfl_up_sync(0xffffffffu, r, 1);
                if (wr) dxc[(long long)c * HW + (long long)y * a.W] = v;
            }
        }
    };

    for (int kc = 0; kc < nch; kc++) {
        const int c0 = kc * CH, cn = min(CH, a.C - c0);
        if (kc + 1 < nch) {
            if (FQ > 0)
                stage_rows<VEC>(stage + ((kc + 1) & 1) * kBStage, FQ, gbase + (long long)(c0 + CH) * P, P,
                                min(CH, a.C - c0 - CH), RQ, a.Wo, ilo, qxa, qoff, qcnt);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *S = stage + (kc & 1) * kBStage;
        switch (cn) {
            case 4: run_chunk(S, c0, std::integral_constant<int, 4>{}); break;
            case 3: run_chunk(S, c0, std::integral_constant<int, 3>{}); break;
            case 2: run_chunk(S, c0, std::integral_constant<int, 2>{}); break;
            default: run_chunk(S, c0, std::integral_constant<int, 1>{}); break;
        }
        __syncthreads();
    }
    // ---- d_theta partial of the cells this tile owns
#pragma unroll
    for (int k = 0; k < 6; k++) {
        const float v = warp_sum(acc6[k]);
        if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double s = 0.0;
        for (int w = 0; w < kBWarps; w++) s += (double)red[w][threadIdx.x];
        part[threadIdx.x] = s;
    }
}

// ----------------------------------------------------------------- backward: lean cell-owner dX
// d_input only (d_theta comes from stn_out_tile<DTHETA> for every sample).  Same
// ownership as stn_bwd_cell, but every warp walks its own halo cell row (no
// cross-warp carry, no barrier inside the chunk loop) and up to kLCH channels
// share one walk, so the per-(cell row, chunk) overhead is paid C/kLCH times.
constexpr int kLRows = 4;                 // px rows per warp
constexpr int kLTY = kLRows * 8;          // 32 px rows per block
#ifndef RS_LSTAGE
#define RS_LSTAGE 8192
#endif
#ifndef RS_LCH
#define RS_LCH 4
#endif
#ifndef RS_LBUFS
#define RS_LBUFS 1
#endif
constexpr int kLBufs = RS_LBUFS;  // dY stage buffers (1: the other block on the SM overlaps)
constexpr int kLRQMax = 160, kLFQMax = 2304, kLStage = RS_LSTAGE, kLCH = RS_LCH;
constexpr int kLCells = (kBX + 1) * (kLTY + 1);  // the block's floor cells: 32 columns x 33 rows
// stage completion: 1 = the stage mbarrier (try_wait spin: ~11% of the kernel's
// instructions, but not of its time), 0 = cp.async groups + a block barrier (measured
// equal: 6.566 vs 6.562 ms for stn_bwd at 64 x 16 x 1024^2)
#ifndef RS_LEAN_MBAR
#define RS_LEAN_MBAR 1
#endif
#ifndef RS_LEAN_RRU
#define RS_LEAN_RRU 5  // full unroll of the 5 cell rows: 6.42 vs 6.55 ms (2: 6.61)
#endif
constexpr int kLRRU = RS_LEAN_RRU;  // unroll of the lean walk's cell-row loop
#ifndef RS_LEAN_FXY
#define RS_LEAN_FXY 1
#endif
#ifndef RS_LEAN_ROWMAX
#define RS_LEAN_ROWMAX 1
#endif
constexpr int kLXT = 256;  // lean: per-block table of the preimage columns' normalised coordinates
constexpr int kLRTot = 8 * (kLRows + 1) > kLTY + 3 ? 8 * (kLRows + 1) : kLTY + 3;

RS_DEV bool stn_lean_ok(const Affine &A, int Ho, int Wo) {
    if (!A.inv || Ho > 65535 || Wo > 65535) return false;
    const double hq = fabs(A.i10) * (kBX + 1) + fabs(A.i11) * (kLTY + 1);
    const double rq = ceil(hq) + 3.0;
    const double fq = (double)(kBX + 1) * (kLTY + 1) / fabs(A.det) + 8.0 * rq + 64.0;
    const double wj = fabs(A.i00) + fabs(A.i01), wi = fabs(A.i10) + fabs(A.i11);
    return rq <= kLRQMax && fq <= kLFQMax && (wj + 2.0) * (wi + 2.0) <= 16.0;
}


// three blocks per SM (76 registers, 32 KB dY stage of 4 channels): 6.64 vs 7.01 ms for
// stn_bwd at 64 x 16 x 1024^2 with two blocks and a 64 KB stage of 8 channels
#ifndef RS_LMINB
#define RS_LMINB 3
#endif
template <bool VEC, bool SELF = false>
__global__ void __launch_bounds__(kThreads, RS_LMINB)
    stn_bwd_lean(StnArgs a, const double *__restrict__ xtab, const double *__restrict__ ytab,
                 const int *__restrict__ flags, int tiles_x, int tiles_y, unsigned *__restrict__ det_slots = nullptr) {
    extern __shared__ __align__(16) float4 sm4[];
    float *stage = (float *)sm4;                               // kLBufs * kLStage
    uint2 *rec = (uint2 *)(stage + kLBufs * kLStage);          // kLFQMax
    int4 *rowt = (int4 *)(rec + kLFQMax);                      // kLRQMax
    int *qlo = (int *)(rowt + kLRQMax);
    int *qhi = qlo + kLRQMax;
    int *qxa = qhi + kLRQMax;
    int *qoff = qxa + kLRQMax;
    int *qcnt = qoff + kLRQMax;
    int *ctl = qcnt + kLRQMax;                                  // 8
    int *cstart = ctl + 8;                                      // kLCells: first hit of each cell
    int *cfill = cstart + kLCells;                              // kLCells: hit counts, then fill ends
    int *rtot = cfill + kLCells;                                // kLRTot: cell row totals, then warp row hit maxima
    unsigned short *hits = (unsigned short *)(rtot + kLRTot);   // kLFQMax: record indices, by cell
    double *xts = (double *)(((uintptr_t)(hits + kLFQMax) + 7) & ~(uintptr_t)7);  // kLXT column coordinates
    __shared__ unsigned long long bars[2];  // stage completion (cp.async.mbarrier.arrive), one per stage

    const int n = blockIdx.y;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int xa0 = tx * kBX, yb0 = ty * kLTY;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long HW = (long long)a.H * a.W, P = (long long)a.Ho * a.Wo;
    const int px = xa0 - 1 + lane;
    float *dxn = a.dx + (long long)n * a.C * HW;
    if (det_slots && blockIdx.x == 0 && blockIdx.y == 0)  // (SELF) the tail's det.cuh slots
        for (int e = threadIdx.x; e < a.N + 2; e += kThreads) det_slots[e] = 0u;
    const Theta T = load_theta(a.theta, n);
    const Affine A = stn_affine(T, a.H, a.W, a.Ho, a.Wo, a.ac);
    // SELF (no prep launch): the block classifies its sample itself (the same test stn_prep makes)
    if (SELF ? !stn_lean_ok(A, a.Ho, a.Wo) : !flags[n]) {  // fallback sample: zero this tile (the atomic scatter adds later)
        if (lane >= 1 && px < a.W)
            for (int r = warp; r < kLTY; r += 8) {
                const int y = yb0 + r;
                if (y < a.H)
                    for (int c = 0; c < a.C; c++) dxn[(long long)c * HW + (long long)y * a.W + px] = 0.f;
            }
        return;
    }
    const double eps = 1e-3;
    const double Lx = xa0 - 1 - eps, Ux = xa0 + kBX + eps;
    const double Ly = yb0 - 1 - eps, Uy = yb0 + kLTY + eps;
    double imin = 1e300, imax = -1e300, jmin = 1e300, jmax = -1e300;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const double px_ = (c & 1) ? Ux : Lx, py_ = (c & 2) ? Uy : Ly;
        const double qi = A.i10 * (px_ - A.p0x) + A.i11 * (py_ - A.p0y);
        imin = fmin(imin, qi);
        imax = fmax(imax, qi);
        if (SELF) {
            const double qj = A.i00 * (px_ - A.p0x) + A.i01 * (py_ - A.p0y);
            jmin = fmin(jmin, qj);
            jmax = fmax(jmax, qj);
        }
    }
    const int ilo = max(0, (int)ceil(fmax(imin, -1e9)));
    const int ihi = min(a.Ho - 1, (int)floor(fmin(imax, 1e9)));
    const int RQ = min(kLRQMax, max(0, ihi - ilo + 1));
    // SELF: the normalised coordinates of the preimage's columns once per block (one
    // division each) instead of a table from the prep launch
    int jlo = 0, jn = 0;
    if (SELF) {
        jlo = max(0, (int)floor(fmax(jmin, -1e9)) - 4);
        jn = min(a.Wo - 1, (int)ceil(fmin(jmax, 1e9)) + 4) - jlo + 1;
        if (jn > kLXT) jn = 0;  // (then stn_norm per record)
        for (int q = threadIdx.x; q < jn; q += kThreads) xts[q] = stn_norm(jlo + q, a.Wo, a.ac);
    }
    for (int r = threadIdx.x; r < RQ; r += kThreads) {
        const int i = ilo + r;
        double jl = -1e300, jh = 1e300;
        const double ax_[2] = {A.m00, A.m10}, bx_[2] = {A.m01 * i + A.p0x, A.m11 * i + A.p0y};
        const double L_[2] = {Lx, Ly}, U_[2] = {Ux, Uy};
#pragma unroll
        for (int d = 0; d < 2; d++) {
            if (fabs(ax_[d]) < 1e-12) {
                if (bx_[d] < L_[d] || bx_[d] > U_[d]) { jl = 1e300; jh = -1e300; }
            } else {
                double u = (L_[d] - bx_[d]) / ax_[d], v = (U_[d] - bx_[d]) / ax_[d];
                if (u > v) { const double t = u; u = v; v = t; }
                jl = fmax(jl, u);
                jh = fmin(jh, v);
            }
        }
        qlo[r] = max(0, (int)ceil(fmax(jl, -1e9)));
        qhi[r] = min(a.Wo - 1, (int)floor(fmin(jh, 1e9)));
    }
    for (int e = threadIdx.x; e < kLCells; e += kThreads) cfill[e] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], kThreads);
        mbar_init(&bars[1], kThreads);
        fence_mbar_init();
    }
    __syncthreads();
    build_rows<VEC>(RQ, a.Wo, qlo, qhi, qxa, qoff, qcnt, &ctl[0]);
    __syncthreads();
    sum_rows(RQ, qcnt, &ctl[1]);
    const int FQ = min(ctl[0], kLFQMax);
    for (int r = threadIdx.x; r < RQ; r += kThreads) rowt[r] = make_int4(qlo[r], qhi[r], qoff[r] - qxa[r], 0);
    for (int r = warp; r < RQ; r += 8) {
        const int i = ilo + r;
        const double yt = SELF ? stn_norm(i, a.Ho, a.ac) : ytab[i];
        const int wr = (qcnt[r] + 3) & ~3;
        for (int col = lane; col < wr; col += 32) {
            const int j = qxa[r] + col, e = qoff[r] + col;
            if (e >= kLFQMax) break;
            uint2 R = make_uint2(0xff000000u, 0xff000000u);
            if (col < qcnt[r] && j >= qlo[r] && j <= qhi[r]) {
                double ix, iy;
                const double xt = !SELF ? xtab[j] : (j - jlo >= 0 && j - jlo < jn) ? xts[j - jlo] : stn_norm(j, a.Wo, a.ac);
                stn_coord(T, xt, yt, a.H, a.W, a.ac, ix, iy);
                const Cell cx = cell_of(ix), cy = cell_of(iy);
                const int rx = cx.i0 - (xa0 - 1), ry = cy.i0 - (yb0 - 1);
                if (rx >= 0 && rx <= kBX && ry >= 0 && ry <= kLTY) R = pack_rec(rx, ry, cx.f, cy.f);
            }
            rec[e] = R;
        }
    }
    const int CH = min(min(a.C, kLCH), FQ > 0 ? max(1, kLStage / FQ) : kLCH);
    const int nch = (a.C + CH - 1) / CH;
    const float *gbase = a.dy + (long long)n * a.C * P;
    __syncthreads();
    // VEC: 16-B cp.async rows completing on the stage's mbarrier; else 4-B cp.async
    auto issue = [&](float *dst, int c0s, int ncp, int slot) {
        if (VEC && RS_LEAN_MBAR) {
            if (FQ > 0) stage_rows<true>(dst, FQ, gbase + (long long)c0s * P, P, ncp, RQ, a.Wo, ilo, qxa, qoff, qcnt);
            cp_async_arrive(&bars[slot]);
        } else {
            if (FQ > 0) stage_rows<VEC>(dst, FQ, gbase + (long long)c0s * P, P, ncp, RQ, a.Wo, ilo, qxa, qoff, qcnt);
            cp_async_commit();
        }
    };
    issue(stage, 0, min(CH, a.C), 0);

    // Per-cell hit lists (CSR over the block's 32 x 33 floor cells): count the records of
    // every cell, scan, place, and sort each short list by record index -- the output
    // pixels of a cell in row-major order, the order the walk sums them in.  (Replaces a
    // per-lane candidate search over the inverse-map window of each cell.)
    for (int e = threadIdx.x; e < FQ; e += kThreads) {
        const uint2 R = rec[e];
        const unsigned rx = R.x >> 24, ry = R.y >> 24;
        if (rx <= (unsigned)kBX && ry <= (unsigned)kLTY) atomicAdd(&cfill[ry * (kBX + 1) + rx], 1);
    }
    __syncthreads();
    for (int ry = warp; ry <= kLTY; ry += 8) {  // exclusive scan within each cell row
        const int v = cfill[ry * 32 + lane];
        int t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        cstart[ry * 32 + lane] = t - v;
        if (lane == 31) rtot[ry] = t;
    }
    __syncthreads();
    if (warp == 0) {  // row bases: exclusive scan of the 33 row totals
        const int v0 = rtot[lane];
        int t = v0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        __syncwarp();
        rtot[lane] = t - v0;
        if (lane == 31) rtot[32] = t;  // row 32 starts after rows 0..31
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kLCells; c += kThreads) {
        const int v = cstart[c] + rtot[c >> 5];
        cstart[c] = v;
        cfill[c] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < FQ; e += kThreads) {
        const uint2 R = rec[e];
        const unsigned rx = R.x >> 24, ry = R.y >> 24;
        if (rx <= (unsigned)kBX && ry <= (unsigned)kLTY) hits[atomicAdd(&cfill[ry * (kBX + 1) + rx], 1)] = (unsigned short)e;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kLCells; c += kThreads) {
        const int b = cstart[c], m = cfill[c] - b;
        for (int i = 1; i < m; i++) {
            const unsigned short key = hits[b + i];
            int j = i - 1;
            while (j >= 0 && hits[b + j] > key) {
                hits[b + j + 1] = hits[b + j];
                j--;
            }
            hits[b + j + 1] = key;
        }
    }
    __syncthreads();
    // the walk reads a hit's fractions in list order: (fx, fy) as float2 at its list
    // position, over the records (no longer needed), and each warp row's maximum hit
    // count once (the walk runs every cell row once per channel chunk)
    {
        const int nh = cfill[kLCells - 1];
        float2 fr[(kLFQMax + kThreads - 1) / kThreads];
#pragma unroll
        for (int k = 0; k < (kLFQMax + kThreads - 1) / kThreads; k++) {
            const int pos = threadIdx.x + k * kThreads;
            if (pos < nh) {
                const uint2 R = rec[hits[pos]];
                fr[k] = make_float2((float)(R.x & 0xffffffu) * (1.f / 16777216.f),
                                    (float)(R.y & 0xffffffu) * (1.f / 16777216.f));
            }
        }
        for (int rr = 0; rr <= kLRows; rr++) {
            const int cell = (kLRows * warp + rr) * (kBX + 1) + lane;
            const int m = __reduce_max_sync(0xffffffffu, cfill[cell] - cstart[cell]);
            if (lane == 0) rtot[warp * (kLRows + 1) + rr] = m;  // (row totals no longer needed)
        }
        __syncthreads();
        float2 *fxy = (float2 *)rec;
#pragma unroll
        for (int k = 0; k < (kLFQMax + kThreads - 1) / kThreads; k++) {
            const int pos = threadIdx.x + k * kThreads;
            if (RS_LEAN_FXY && pos < nh) fxy[pos] = fr[k];
        }
    }
    __syncthreads();
    const float2 *fxy = (const float2 *)rec;
    const uint2 *recs = rec;
    const int *rowmax = rtot + warp * (kLRows + 1);

    // every warp walks its own halo cell row: rows wy0-1 .. wy0+kLRows-1 (cell rows
    // 4 warp .. 4 warp + 4 of the block; lane = cell column)
    const int wy0 = yb0 + kLRows * warp;
    const bool pxin = lane >= 1 && px < a.W;

    auto run_chunk = [&](const float *S, int c0, auto ncc) {
        constexpr int NC = decltype(ncc)::value;
        float L[NC], Rr[NC], NL[NC], NR[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) NL[c] = NR[c] = 0.f;
        float *drow = dxn + (long long)c0 * HW + (long long)(wy0 - 1) * a.W + px;
#pragma unroll (kLRRU)
        for (int rr = 0; rr <= kLRows; rr++, drow += a.W) {
            const int y0 = wy0 - 1 + rr;
#pragma unroll
            for (int c = 0; c < NC; c++) { L[c] = NL[c]; Rr[c] = NR[c]; NL[c] = 0.f; NR[c] = 0.f; }
            auto process = [&](int pos) {
                const int e = hits[pos];
#if RS_LEAN_FXY
                const float2 f = fxy[pos];
                const float fx = f.x, fy = f.y;
#else
                const uint2 R = recs[e];
                const float fx = (float)(R.x & 0xffffffu) * (1.f / 16777216.f);
                const float fy = (float)(R.y & 0xffffffu) * (1.f / 16777216.f);
#endif
                const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
                const float w10 = fy * (1.f - fx), w11 = fy * fx;
                const float *Se = S + e;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const float g = Se[c * FQ];
                    L[c] = fmaf(w00, g, L[c]);
                    Rr[c] = fmaf(w01, g, Rr[c]);
                    NL[c] = fmaf(w10, g, NL[c]);
                    NR[c] = fmaf(w11, g, NR[c]);
                }
            };
            const int cell = (kLRows * warp + rr) * (kBX + 1) + lane;
            const int hb = cstart[cell], hn = cfill[cell] - hb;
#if RS_LEAN_ROWMAX
            const int hmax = rowmax[rr];
#else
            const int hmax = __reduce_max_sync(0xffffffffu, hn);
#endif
            for (int h = 0; h < hmax; h++)
                if (h < hn) process(hb + h);
            if (rr > 0) {  // row 0 is the halo: it only seeds the carry
                const bool wr = pxin && y0 < a.H;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const float v = L[c] + __shfl_up_sync(0xffffffffu, Rr[c], 1);
                    if (wr) drow[(long long)c * HW] = v;
                }
            }
        }
    };

    for (int kc = 0; kc < nch; kc++) {
        const int c0 = kc * CH, cn = min(CH, a.C - c0);
        if (kLBufs == 2 && kc + 1 < nch)
            issue(stage + ((kc + 1) % kLBufs) * kLStage, c0 + CH, min(CH, a.C - c0 - CH), (kc + 1) & 1);
        if (VEC && RS_LEAN_MBAR) {
            mbar_wait(&bars[kc & 1], (unsigned)((kc >> 1) & 1));
            if (RS_RACECHECK_SYNC) {
                cp_async_wait<0>();
                __syncthreads();
            }
        } else {
            if (kLBufs == 2 && kc + 1 < nch) cp_async_wait<1>();
            else cp_async_wait<0>();
        }
        if (!(VEC && RS_LEAN_MBAR)) __syncthreads();
        const float *S = stage + (kc % kLBufs) * kLStage;
        switch (cn) {
            case 8: run_chunk(S, c0, std::integral_constant<int, 8>{}); break;
            case 7: run_chunk(S, c0, std::integral_constant<int, 7>{}); break;
            case 6: run_chunk(S, c0, std::integral_constant<int, 6>{}); break;
            case 5: run_chunk(S, c0, std::integral_constant<int, 5>{}); break;
            case 4: run_chunk(S, c0, std::integral_constant<int, 4>{}); break;
            case 3: run_chunk(S, c0, std::integral_constant<int, 3>{}); break;
            case 2: run_chunk(S, c0, std::integral_constant<int, 2>{}); break;
            default: run_chunk(S, c0, std::integral_constant<int, 1>{}); break;
        }
        __syncthreads();
        if (kLBufs == 1 && kc + 1 < nch) issue(stage, c0 + CH, min(CH, a.C - c0 - CH), (kc + 1) & 1);
    }
}

// ----------------------------------------------------------------- backward: per-pixel gather
// Input tile 32 x 16 (thread = column, rows w and w+8).  Each input pixel p walks
// the preimage window of [p-1, p+1)^2 once, keeping its (<= kGHits) hits — the
// output pixels whose floor cell is p-(0|1) — as (record index, weight); every
// channel chunk then costs one LDS + FMA per hit.  dY over the tile's preimage
// and X over the tile (+1 halo) are staged per chunk (cp.async, double-buffered).
// d_theta: pixel p owns the hits whose floor cell is p (x0 = -1 folds into x = 0).
constexpr int kGX = 32, kGY = 16, kGHits = 8;
constexpr int kGXP = kGX + 4;            // X stage pitch (16-B rows)
constexpr int kGXS = (kGY + 1) * kGXP;   // X stage floats per channel
constexpr int kGRQMax = 128, kGFQMax = 1792, kGStage = 8192, kGCH = 4;

RS_DEV bool stn_gather_ok(const Affine &A, int Ho, int Wo) {
    if (!A.inv || Ho > 65535 || Wo > 65535) return false;
    const double hq = fabs(A.i10) * (kGX + 1) + fabs(A.i11) * (kGY + 1);
    const double rq = ceil(hq) + 3.0;
    const double fq = (double)(kGX + 1) * (kGY + 1) / fabs(A.det) + 8.0 * rq + 64.0;
    const double wj = fabs(A.i00) + fabs(A.i01), wi = fabs(A.i10) + fabs(A.i11);
    return rq <= kGRQMax && fq <= kGFQMax && (2.0 * wj + 2.0) * (2.0 * wi + 2.0) <= 36.0;
}

template <bool VEC>
__global__ void __launch_bounds__(kThreads, 2)
    stn_bwd_gather(StnArgs a, const double *__restrict__ xtab, const double *__restrict__ ytab,
                   const int *__restrict__ flags, double *__restrict__ partials, int tiles_x, int tiles_y) {
    extern __shared__ __align__(16) float4 sm4[];
    float *stage = (float *)sm4;                               // 2 * kGStage
    uint2 *rec = (uint2 *)(stage + 2 * kGStage);               // kGFQMax
    unsigned *ijs = (unsigned *)(rec + kGFQMax);               // kGFQMax
    int4 *rowt = (int4 *)(ijs + kGFQMax);                      // kGRQMax
    int *qlo = (int *)(rowt + kGRQMax);
    int *qhi = qlo + kGRQMax;
    int *qxa = qhi + kGRQMax;
    int *qoff = qxa + kGRQMax;
    int *qcnt = qoff + kGRQMax;
    int *ctl = qcnt + kGRQMax;                                  // 8
    __shared__ float red[kThreads / 32][6];

    const int n = blockIdx.y;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int xa0 = tx * kGX, ya0 = ty * kGY;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long HW = (long long)a.H * a.W, P = (long long)a.Ho * a.Wo;
    const int x = xa0 + lane;
    float *dxn = a.dx ? a.dx + (long long)n * a.C * HW : nullptr;
    double *part = partials + ((long long)n * tiles_x * tiles_y + blockIdx.x) * 6;

    if (!flags[n]) {
        if (dxn && x < a.W)
            for (int r = warp; r < kGY; r += 8) {
                const int y = ya0 + r;
                if (y < a.H)
                    for (int c = 0; c < a.C; c++) dxn[(long long)c * HW + (long long)y * a.W + x] = 0.f;
            }
        if (threadIdx.x < 6) part[threadIdx.x] = 0.0;
        return;
    }
    const Theta T = load_theta(a.theta, n);
    const Affine A = stn_affine(T, a.H, a.W, a.Ho, a.Wo, a.ac);

    // ---- preimage rows of the cells [xa0-1, xa0+kGX-1] x [ya0-1, ya0+kGY-1]
    const double eps = 1e-3;
    const double Lx = xa0 - 1 - eps, Ux = xa0 + kGX + eps;
    const double Ly = ya0 - 1 - eps, Uy = ya0 + kGY + eps;
    double imin = 1e300, imax = -1e300;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const double px_ = (c & 1) ? Ux : Lx, py_ = (c & 2) ? Uy : Ly;
        const double qi = A.i10 * (px_ - A.p0x) + A.i11 * (py_ - A.p0y);
        imin = fmin(imin, qi);
        imax = fmax(imax, qi);
    }
    const int ilo = max(0, (int)ceil(fmax(imin, -1e9)));
    const int ihi = min(a.Ho - 1, (int)floor(fmin(imax, 1e9)));
    const int RQ = min(kGRQMax, max(0, ihi - ilo + 1));
    for (int r = threadIdx.x; r < RQ; r += kThreads) {
        const int i = ilo + r;
        double jl = -1e300, jh = 1e300;
        const double ax_[2] = {A.m00, A.m10}, bx_[2] = {A.m01 * i + A.p0x, A.m11 * i + A.p0y};
        const double L_[2] = {Lx, Ly}, U_[2] = {Ux, Uy};
#pragma unroll
        for (int d = 0; d < 2; d++) {
            if (fabs(ax_[d]) < 1e-12) {
                if (bx_[d] < L_[d] || bx_[d] > U_[d]) { jl = 1e300; jh = -1e300; }
            } else {
                double u = (L_[d] - bx_[d]) / ax_[d], v = (U_[d] - bx_[d]) / ax_[d];
                if (u > v) { const double t = u; u = v; v = t; }
                jl = fmax(jl, u);
                jh = fmin(jh, v);
            }
        }
        qlo[r] = max(0, (int)ceil(fmax(jl, -1e9)));
        qhi[r] = min(a.Wo - 1, (int)floor(fmin(jh, 1e9)));
    }
    __syncthreads();
    build_rows<VEC>(RQ, a.Wo, qlo, qhi, qxa, qoff, qcnt, &ctl[0]);
    __syncthreads();
    const int FQ = min(ctl[0], kGFQMax);
    for (int r = threadIdx.x; r < RQ; r += kThreads) rowt[r] = make_int4(qlo[r], qhi[r], qoff[r] - qxa[r], 0);
    for (int r = warp; r < RQ; r += 8) {
        const int i = ilo + r;
        const double yt = ytab[i];
        const int wr = (qcnt[r] + 3) & ~3;
        for (int col = lane; col < wr; col += 32) {
            const int j = qxa[r] + col, e = qoff[r] + col;
            if (e >= kGFQMax) break;
            uint2 R = make_uint2(0xff000000u, 0xff000000u);
            if (col < qcnt[r] && j >= qlo[r] && j <= qhi[r]) {
                double ix, iy;
                stn_coord(T, xtab[j], yt, a.H, a.W, a.ac, ix, iy);
                const Cell cx = cell_of(ix), cy = cell_of(iy);
                const int rx = cx.i0 - (xa0 - 1), ry = cy.i0 - (ya0 - 1);
                if (rx >= 0 && rx <= kGX && ry >= 0 && ry <= kGY) R = pack_rec(rx, ry, cx.f, cy.f);
            }
            rec[e] = R;
            ijs[e] = ((unsigned)i << 16) | (unsigned)j;
        }
    }
    const int XS = kGXS;
    const int CH = min(min(a.C, kGCH), max(1, kGStage / (FQ + XS)));
    const int nch = (a.C + CH - 1) / CH;
    const float *gbase = a.dy + (long long)n * a.C * P;
    const float *xbase = a.x + (long long)n * a.C * HW;
    const bool xvec = VEC && (a.W % 4 == 0) && (((uintptr_t)a.x & 15u) == 0);
    // X stage: rows ya0..ya0+kGY, columns [xa0, xa0 + kGXP) clipped to the image
    auto stage_x = [&](float *dst, int c0, int ncp) {
        const int cw = min(kGXP, a.W - xa0);
        for (int e = threadIdx.x; e < ncp * (kGY + 1); e += kThreads) {
            const int c = e / (kGY + 1), r = e - c * (kGY + 1);
            const int y = ya0 + r;
            if (y >= a.H) continue;
            const float *src = xbase + (long long)(c0 + c) * HW + (long long)y * a.W + xa0;
            float *d = dst + c * XS + r * kGXP;
            if (xvec) {
                for (int q = 0; q < cw; q += 4) cp_async16(d + q, src + q);
            } else {
                for (int q = 0; q < cw; q++) cp_async4(d + q, src + q);
            }
        }
    };
    __syncthreads();
    if (FQ > 0) stage_rows<VEC>(stage, FQ, gbase, P, min(CH, a.C), RQ, a.Wo, ilo, qxa, qoff, qcnt);
    stage_x(stage + CH * FQ, 0, min(CH, a.C));
    cp_async_commit();

    // ---- per-pixel hit lists (overlaps the first stage's copy)
    const double hj = fabs(A.i00) + fabs(A.i01) + eps, hi = fabs(A.i10) + fabs(A.i11) + eps;
    // fn(e, weight, hit index) for every output pixel that samples this pixel;
    // also reports whether the pixel owns it (floor cell == pixel, -1 folded to 0)
    auto search = [&](int k, auto &&fn) {
        const int y = ya0 + warp + 8 * k;
        const double ux = (double)x - A.p0x, uy = (double)y - A.p0y;
        const double qj = A.i00 * ux + A.i01 * uy, qi = A.i10 * ux + A.i11 * uy;
        const int jl = (int)ceil(qj - hj), jh = (int)floor(qj + hj);
        const int il = max(ilo, (int)ceil(qi - hi)), ih = min(ilo + RQ - 1, (int)floor(qi + hi));
        const unsigned rx0 = (unsigned)(x - (xa0 - 1)), ry0 = (unsigned)(y - (ya0 - 1));
        int cnt = 0;
        for (int i = il; i <= ih; i++) {
            const int4 rt = rowt[i - ilo];
            const int ja = max(jl, rt.x), jb = min(jh, rt.y);
            for (int j = ja; j <= jb; j++) {
                const int e = rt.z + j;
                const uint2 R = rec[e];
                const unsigned rx = R.x >> 24, ry = R.y >> 24;
                if ((rx == rx0 || rx + 1 == rx0) && (ry == ry0 || ry + 1 == ry0)) {
                    const float fx = (float)(R.x & 0xffffffu) * (1.f / 16777216.f);
                    const float fy = (float)(R.y & 0xffffffu) * (1.f / 16777216.f);
                    const float wx = (rx == rx0) ? 1.f - fx : fx, wy = (ry == ry0) ? 1.f - fy : fy;
                    fn(e, wy * wx, cnt);
                    cnt++;
                }
            }
        }
        return cnt;
    };
    int he[2][kGHits];
    float hw[2][kGHits];
    int nh[2];
    unsigned own[2];
    bool pin[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const int y = ya0 + warp + 8 * k;
        pin[k] = x < a.W && y < a.H;
        nh[k] = 0;
        own[k] = 0u;
#pragma unroll
        for (int h = 0; h < kGHits; h++) { he[k][h] = 0; hw[k][h] = 0.f; }
        if (!pin[k]) continue;
        nh[k] = search(k, [&](int e, float w, int cnt) {
#pragma unroll
            for (int h = 0; h < kGHits; h++)
                if (h == cnt) { he[k][h] = e; hw[k][h] = w; }
            const uint2 R = rec[e];
            const int x0 = (int)(R.x >> 24) + xa0 - 1, y0 = (int)(R.y >> 24) + ya0 - 1;
            // the pixel owns the output pixels whose floor cell it is (-1 folded to 0);
            // owned hits always fit the cache: at most the first kGHits are owned-tracked
            if (max(x0, 0) == x && max(y0, 0) == y && cnt < kGHits) own[k] |= 1u << cnt;
        });
    }
    float acc6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float sxs = a.ac ? 0.5f * (a.W - 1) : 0.5f * a.W;
    const float sys = a.ac ? 0.5f * (a.H - 1) : 0.5f * a.H;
    const float axf = a.ac ? 2.f / (a.Wo - 1) : 2.f / a.Wo, bxf = a.ac ? -1.f : 1.f / a.Wo - 1.f;
    const float ayf = a.ac ? 2.f / (a.Ho - 1) : 2.f / a.Ho, byf = a.ac ? -1.f : 1.f / a.Ho - 1.f;

    auto run_chunk = [&](const float *S, int c0, auto ncc) {
        constexpr int NC = decltype(ncc)::value;
        const float *SX = S + CH * FQ;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int y = ya0 + warp + 8 * k;
            const bool ovf = pin[k] && nh[k] > kGHits;
            float acc[NC];
#pragma unroll
            for (int c = 0; c < NC; c++) acc[c] = 0.f;
            const int hmax = __reduce_max_sync(0xffffffffu, pin[k] ? min(nh[k], kGHits) : 0);
#pragma unroll
            for (int h = 0; h < kGHits; h++) {
                if (h < hmax && h < nh[k]) {
                    const float *Se = S + he[k][h];
#pragma unroll
                    for (int c = 0; c < NC; c++) acc[c] = fmaf(hw[k][h], Se[c * FQ], acc[c]);
                }
            }
            // d_theta of the output pixels this pixel owns (floor cell == this pixel)
            if (own[k] || ovf) {
                float dxa[NC], ddx[NC], dya[NC], ddy[NC];
                const float *X0 = SX + (y - ya0) * kGXP + (x - xa0);
                const bool xv1 = x + 1 < a.W, yv1 = y + 1 < a.H;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const float *Xc = X0 + c * XS;
                    const float v00 = Xc[0], v01 = xv1 ? Xc[1] : 0.f;
                    const float v10 = yv1 ? Xc[kGXP] : 0.f, v11 = (xv1 && yv1) ? Xc[kGXP + 1] : 0.f;
                    dxa[c] = v01 - v00;
                    ddx[c] = (v11 - v10) - dxa[c];
                    dya[c] = v10 - v00;
                    ddy[c] = (v11 - v01) - dya[c];
                }
                auto dtheta_hit = [&](int e) {
                    const uint2 R = rec[e];
                    const float fx = (float)(R.x & 0xffffffu) * (1.f / 16777216.f);
                    const float fy = (float)(R.y & 0xffffffu) * (1.f / 16777216.f);
                    const int x0 = (int)(R.x >> 24) + xa0 - 1, y0 = (int)(R.y >> 24) + ya0 - 1;
                    const float *Se = S + e;
                    float dq = 0.f, dr = 0.f;
#pragma unroll
                    for (int c = 0; c < NC; c++) {
                        const float g = Se[c * FQ];
                        float a0 = dxa[c], a1 = ddx[c], b0 = dya[c], b1 = ddy[c];
                        if (x0 < 0 || y0 < 0) {
                            // edge cell (x0 = -1 and/or y0 = -1, owned by x = 0 / y = 0):
                            // the taps left of / above the image read 0
                            const float *Xc = X0 + c * XS;
                            float w01 = 0.f, w10 = 0.f, w11;
                            if (x0 < 0 && y0 < 0) {
                                w11 = Xc[0];
                            } else if (x0 < 0) {
                                w01 = Xc[0];
                                w11 = yv1 ? Xc[kGXP] : 0.f;
                            } else {
                                w10 = Xc[0];
                                w11 = xv1 ? Xc[1] : 0.f;
                            }
                            a0 = w01;
                            a1 = (w11 - w10) - a0;
                            b0 = w10;
                            b1 = (w11 - w01) - b0;
                        }
                        dq = fmaf(g, fmaf(fy, a1, a0), dq);
                        dr = fmaf(g, fmaf(fx, b1, b0), dr);
                    }
                    const unsigned ij = ijs[e];
                    const float xt = fmaf(axf, (float)(ij & 0xffffu), bxf);
                    const float yt = fmaf(ayf, (float)(ij >> 16), byf);
                    const float dgx = dq * sxs, dgy = dr * sys;
                    acc6[0] = fmaf(dgx, xt, acc6[0]);
                    acc6[1] = fmaf(dgx, yt, acc6[1]);
                    acc6[2] += dgx;
                    acc6[3] = fmaf(dgy, xt, acc6[3]);
                    acc6[4] = fmaf(dgy, yt, acc6[4]);
                    acc6[5] += dgy;
                };
#pragma unroll
                for (int h = 0; h < kGHits; h++)
                    if (own[k] & (1u << h)) dtheta_hit(he[k][h]);
                if (ovf) {
                    // more hits than cached: walk the window again for the rest (rare)
                    search(k, [&](int e, float w, int idx) {
                        if (idx < kGHits) return;
                        const float *Se = S + e;
#pragma unroll
                        for (int c = 0; c < NC; c++) acc[c] = fmaf(w, Se[c * FQ], acc[c]);
                        const uint2 R = rec[e];
                        const int x0 = (int)(R.x >> 24) + xa0 - 1, y0 = (int)(R.y >> 24) + ya0 - 1;
                        if (max(x0, 0) == x && max(y0, 0) == y) dtheta_hit(e);
                    });
                }
            }
            if (dxn && pin[k]) {
                float *d = dxn + (long long)c0 * HW + (long long)y * a.W + x;
#pragma unroll
                for (int c = 0; c < NC; c++) d[(long long)c * HW] = acc[c];
            }
        }
    };

    for (int kc = 0; kc < nch; kc++) {
        const int c0 = kc * CH, cn = min(CH, a.C - c0);
        if (kc + 1 < nch) {
            float *nxt = stage + ((kc + 1) & 1) * kGStage;
            const int cn2 = min(CH, a.C - c0 - CH);
            if (FQ > 0) stage_rows<VEC>(nxt, FQ, gbase + (long long)(c0 + CH) * P, P, cn2, RQ, a.Wo, ilo, qxa, qoff, qcnt);
            stage_x(nxt + CH * FQ, c0 + CH, cn2);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *S = stage + (kc & 1) * kGStage;
        switch (cn) {
            case 4: run_chunk(S, c0, std::integral_constant<int, 4>{}); break;
            case 3: run_chunk(S, c0, std::integral_constant<int, 3>{}); break;
            case 2: run_chunk(S, c0, std::integral_constant<int, 2>{}); break;
            default: run_chunk(S, c0, std::integral_constant<int, 1>{}); break;
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 6; k++) {
        const float v = warp_sum(acc6[k]);
        if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; w++) s += (double)red[w][threadIdx.x];
        part[threadIdx.x] = s;
    }
}

// ----------------------------------------------------------------- d_theta finalize
// dtheta[n] = fixed-order fp64 sum of the partials of the path sample n took.
__global__ void __launch_bounds__(kThreads)
    stn_dtheta_finalize(const double *__restrict__ pb, int nb, const double *__restrict__ pf, int nf,
                        const int *__restrict__ flags, float *dtheta) {
    const int n = blockIdx.x;
    const bool g = flags ? flags[n] != 0 : false;  // flags == nullptr: every sample used the output tiles
    const double *p = g ? pb + (long long)n * nb * 6 : pf + (long long)n * nf * 6;
    const int nt = g ? nb : nf;
    __shared__ double red[kThreads / 32][6];
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nt; b += kThreads)
#pragma unroll
        for (int k = 0; k < 6; k++) s[k] += p[(long long)b * 6 + k];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; k++) {
        const double v = warp_sum_d(s[k]);
        if (lane == 0) red[wid][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = 0.0;
        for (int w = 0; w < kThreads / 32; w++) v += red[w][threadIdx.x];
        dtheta[6 * n + threadIdx.x] = (float)v;
    }
}

// ----------------------------------------------------------------- atomic scatter (fallback samples)
// A fallback sample whose map gathers many output pixels onto one input cell (a singular
// map, or a zoom-out with 4 / |det| > 64 output pixels per input pixel) would sum hundreds
// to thousands of fp32 reds per element: with cancelling terms beyond the north star's
// gradient tolerance, as the warp layer's collapsing flows were.  Such "heavy" samples
// take the fixed-point scatter (det.cuh), exact to ~1e-11, in AUTO as well.
RS_DEV bool stn_heavy(const Affine &A, int border = 0, int H = 0, int W = 0, int Ho = 0, int Wo = 0) {
    if (!A.inv || fabs(A.det) < 4.0 / 64.0) return true;
    if (!border) return false;
    // border padding clamps every tap outside the image onto its edge (a corner pixel
    // collects the whole region beyond both edges): heavy once the output reaches outside
    for (int c = 0; c < 4; c++) {
        const double qx = (c & 1) ? Wo - 1 : 0, qy = (c & 2) ? Ho - 1 : 0;
        const double px = A.p0x + A.m00 * qx + A.m01 * qy, py = A.p0y + A.m10 * qx + A.m11 * qy;
        if (px < -1.0 || px > W || py < -1.0 || py > H) return true;
    }
    return false;
}

__global__ void __launch_bounds__(kThreads)
    stn_dx_scatter(StnArgs a, const int *__restrict__ fb_list, const int *__restrict__ fb_count) {
    const long long P = (long long)a.Ho * a.Wo, HW = (long long)a.H * a.W;
    const int nf = *fb_count;
    for (int f = 0; f < nf; f++) {
        const int n = fb_list[f];
        const Theta T = load_theta(a.theta, n);
        if (stn_heavy(stn_affine(T, a.H, a.W, a.Ho, a.Wo, a.ac), a.border, a.H, a.W, a.Ho, a.Wo)) continue;  // (fixed-point scatter)
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
            if (!((x0ok || x1ok) && (y0ok || y1ok))) continue;
            const float w00 = (1.f - cy.f) * (1.f - cx.f), w01 = (1.f - cy.f) * cx.f;
            const float w10 = cy.f * (1.f - cx.f), w11 = cy.f * cx.f;
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
}

// Bilinear STN taps for the deterministic fixed-point scatter (det.cuh): the same
// exact fp64 coordinate and fp32 weights as stn_dx_scatter.
struct StnTapSampler {
    const float *theta;
    int H, W, Ho, Wo, ac, border;
    static constexpr int kMaxTaps = 4;
    static constexpr double kWmax = 1.0;
    RS_DEV int taps(int n, long long q, long long *off, float *w) const {
        const int i = (int)(q / Wo), j = (int)(q - (long long)i * Wo);
        const Theta T = load_theta(theta, n);
        double ix, iy;
        stn_coord(T, stn_norm(j, Wo, ac), stn_norm(i, Ho, ac), H, W, ac, ix, iy);
        if (border) {
            float d;
            ix = clamp_coord(ix, W, d);
            iy = clamp_coord(iy, H, d);
        }
        const Cell cx = cell_of(ix), cy = cell_of(iy);
        const bool x0ok = cx.i0 >= 0 && cx.i0 < W, x1ok = cx.i0 + 1 >= 0 && cx.i0 + 1 < W;
        const bool y0ok = cy.i0 >= 0 && cy.i0 < H, y1ok = cy.i0 + 1 >= 0 && cy.i0 + 1 < H;
        const long long o00 = (long long)cy.i0 * W + cx.i0;
        int k = 0;
        if (y0ok && x0ok) { off[k] = o00; w[k++] = (1.f - cy.f) * (1.f - cx.f); }
        if (y0ok && x1ok) { off[k] = o00 + 1; w[k++] = (1.f - cy.f) * cx.f; }
        if (y1ok && x0ok) { off[k] = o00 + W; w[k++] = cy.f * (1.f - cx.f); }
        if (y1ok && x1ok) { off[k] = o00 + W + 1; w[k++] = cy.f * cx.f; }
        return k;
    }
};

// ----------------------------------------------------------------- lean path tail
// The last launch of the lean backward when no prep kernel ran (cooperative: every block
// co-resident): d_theta of every sample as the fixed-order sum of its tile partials
// (stn_dtheta_finalize's order), then every sample that stn_bwd_lean classified as a
// fallback (singular / huge preimage: its dX tiles were zeroed) gets the exact
// fixed-point scatter of det.cuh -- one launch instead of prep + scatter + finalize.
// ws.maxbits[n] must be zero on entry (stn_bwd_lean<SELF> zeroes them).
__global__ void __launch_bounds__(kThreads)
    stn_det_tail(StnArgs a, const double *__restrict__ pf, int nf, DetWs ws) {
    __shared__ double redd[kThreads / 32][6];
    __shared__ unsigned redu[kThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (a.dtheta)
        for (int n = blockIdx.x; n < a.N; n += gridDim.x) {  // block-uniform
            const double *p = pf + (long long)n * nf * 6;
            double sk[6] = {0, 0, 0, 0, 0, 0};
            for (int b = threadIdx.x; b < nf; b += kThreads)
#pragma unroll
                for (int k = 0; k < 6; k++) sk[k] += p[(long long)b * 6 + k];
#pragma unroll
            for (int k = 0; k < 6; k++) {
                const double v = warp_sum_d(sk[k]);
                if (lane == 0) redd[wid][k] = v;
            }
            __syncthreads();
            if (threadIdx.x < 6) {
                double v = 0.0;
                for (int w = 0; w < kThreads / 32; w++) v += redd[w][threadIdx.x];
                a.dtheta[6 * n + threadIdx.x] = (float)v;
            }
            __syncthreads();
        }
    if (!a.dx) return;
    const StnTapSampler smp{a.theta, a.H, a.W, a.Ho, a.Wo, a.ac, a.border};
    const long long HW = (long long)a.H * a.W, P = (long long)a.Ho * a.Wo;
    for (int m = 0; m < a.N; m++) {
        if (stn_lean_ok(stn_affine(load_theta(a.theta, m), a.H, a.W, a.Ho, a.Wo, a.ac), a.Ho, a.Wo)) continue;
        det_scatter_one<StnTapSampler, kThreads>(smp, a.dy, a.dx, m, m, a.C, HW, P, ws, redu, 1);
    }
}

// ----------------------------------------------------------------- host helpers
size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

struct StnGeom {
    int fj, fi;  // output tiles (d_theta tile rows)
    int fi_fwd;  // output tile rows of the forward
    int bx, by;  // input tiles, cell-owner kernel
    int gx, gy;  // input tiles, per-pixel gather kernel
};

StnGeom stn_geom(int H, int W, int Ho, int Wo) {
    StnGeom g;
    g.fj = (Wo + kFJ - 1) / kFJ;
    g.fi = (Ho + kFIdth - 1) / kFIdth;
    g.fi_fwd = (Ho + kFIfwd - 1) / kFIfwd;
    g.bx = (W + kBX - 1) / kBX;
    g.by = (H + kBTY - 1) / kBTY;
    g.gx = (W + kGX - 1) / kGX;
    g.gy = (H + kGY - 1) / kGY;
    return g;
}

// STN backward variant: 0 = cell-owner (default, measured faster: profiles/), 1 =
// per-pixel gather.  RSGRAD_STN_BWD=cell|gather selects one (A/B measurements);
// read per call so tests can switch.
int stn_bwd_variant() {
    const char *e = getenv("RSGRAD_STN_BWD");
    if (e && strcmp(e, "gather") == 0) return 1;
    if (e && strcmp(e, "cell") == 0) return 0;
    return 2;  // lean dX + staged output-tile d_theta (measured fastest)
}

struct StnWs {
    double *xtab, *ytab, *pb, *pf;
    int *flags, *fb_list, *fb_count, *ctr, *hv_list, *hv_count;
    void *det;  // deterministic fallback scatter (det.cuh), when requested
    size_t bytes;
};

StnWs stn_ws_layout(void *base, int N, int C, int H, int W, int Ho, int Wo, bool det) {
    const StnGeom g = stn_geom(H, W, Ho, Wo);
    StnWs w;
    size_t off = 0;
    char *b = (char *)base;
    auto take = [&](size_t bytes) {
        void *p = b ? b + off : nullptr;
        off += align256(bytes);
        return p;
    };
    w.xtab = (double *)take(sizeof(double) * Wo);
    w.ytab = (double *)take(sizeof(double) * Ho);
    w.flags = (int *)take(sizeof(int) * N);
    w.fb_list = (int *)take(sizeof(int) * N);
    w.fb_count = (int *)take(sizeof(int));
    w.ctr = (int *)take(sizeof(int) * N);
    const size_t tb = (size_t)g.bx * g.by > (size_t)g.gx * g.gy ? (size_t)g.bx * g.by : (size_t)g.gx * g.gy;
    w.pb = (double *)take(sizeof(double) * 6 * (size_t)N * tb);
    w.pf = (double *)take(sizeof(double) * 6 * (size_t)N * g.fj * g.fi);
    w.hv_list = (int *)take(sizeof(int) * N);
    w.hv_count = (int *)take(sizeof(int));
    // fixed-point accumulators: every channel for deterministic=1, one channel plane for
    // AUTO's heavy samples (walked a channel at a time: det_scatter_one's cpp = 1)
    w.det = take(det_ws_bytes(N, (det ? (long long)C : 1LL) * H * W));
    w.bytes = off;
    return w;
}

// RSGRAD_STN_TILES=slow selects the cp.async output-tile path (A/B comparisons)
bool stn_slow_tiles() {
    const char *e = getenv("RSGRAD_STN_TILES");
    return e && strcmp(e, "slow") == 0;
}

size_t out_tile_smem() {
    const int st = 2 * kFStage > kNS * kFSt ? 2 * kFStage : kNS * kFSt;
    return sizeof(int) * (5 * kFRMax + 16) + sizeof(float) * st;
}
size_t bwd_lean_smem() {
    return sizeof(float) * kLBufs * kLStage + sizeof(uint2) * kLFQMax + sizeof(int4) * kLRQMax +
           sizeof(int) * (5 * kLRQMax + 8 + 2 * kLCells + kLRTot) + sizeof(unsigned short) * kLFQMax + 8 +
           sizeof(double) * kLXT;
}

size_t bwd_gather_smem() {
    return sizeof(float) * 2 * kGStage + (sizeof(uint2) + sizeof(unsigned)) * kGFQMax + sizeof(int4) * kGRQMax +
           sizeof(int) * (5 * kGRQMax + 8);
}

size_t bwd_cell_smem() {
    return sizeof(float) * 2 * kBStage + (sizeof(uint2) + sizeof(unsigned)) * kBFQMax +
           sizeof(int4) * kBRQMax + sizeof(int) * (5 * kBRQMax + 8) + sizeof(float) * kBWarps * 2 * kBCH * 32 +
           sizeof(unsigned short) * kBWarps * (kBRows + 1) * kBHits * 32 + kBWarps * (kBRows + 1) * 32;
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

size_t stn_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det) {
    return stn_ws_layout(nullptr, N, C, H, W, Ho, Wo, det).bytes;
}

cudaError_t stn_fwd_launch(const StnArgs &a, cudaStream_t s) {
    const StnGeom g = stn_geom(a.H, a.W, a.Ho, a.Wo);
    const bool vec = (a.W % 4 == 0) && aligned16(a.x);
    const size_t sm = out_tile_smem();
    dim3 grid(g.fj * g.fi_fwd, a.N);
    if (vec && !stn_slow_tiles()) {
        auto k = stn_out_tile<MODE_FWD, true, false, kFIfwd, true>;
        set_smem(k, sm);
        k<<<grid, kOTFast, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr, nullptr, g.fj, g.fi_fwd, nullptr);
    } else if (vec) {
        set_smem(stn_out_tile<MODE_FWD, true>, sm);
        stn_out_tile<MODE_FWD, true><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                nullptr, g.fj, g.fi_fwd);
    } else {
        set_smem(stn_out_tile<MODE_FWD, false>, sm);
        stn_out_tile<MODE_FWD, false><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                 nullptr, g.fj, g.fi_fwd);
    }
    note_launch();
    return cudaGetLastError();
}

cudaError_t flow_tile_launch(const StnArgs &a, int mode, bool priv, cudaStream_t s) {
    const StnGeom g = stn_geom(a.H, a.W, a.Ho, a.Wo);
    const bool vec = (a.W % 4 == 0) && aligned16(a.x);
    const size_t sm = out_tile_smem();
    dim3 grid(g.fj * g.fi, a.N);
    if (mode == MODE_FWD) {
        grid.x = g.fj * g.fi_fwd;
        if (vec) {
            set_smem(stn_out_tile<MODE_FWD, true, true>, sm);
            stn_out_tile<MODE_FWD, true, true><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                          nullptr, g.fj, g.fi_fwd);
        } else {
            set_smem(stn_out_tile<MODE_FWD, false, true>, sm);
            stn_out_tile<MODE_FWD, false, true><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                           nullptr, g.fj, g.fi_fwd);
        }
    } else if (priv) {
        const size_t smp = sm + sizeof(float) * kFStage;
        if (vec) {
            auto k = stn_out_tile<MODE_DFLOW, true, true, kFIdth, false, true>;
            set_smem(k, smp);
            k<<<grid, kThreads, smp, s>>>(a, nullptr, nullptr, nullptr, nullptr, nullptr, g.fj, g.fi, nullptr);
        } else {
            auto k = stn_out_tile<MODE_DFLOW, false, true, kFIdth, false, true>;
            set_smem(k, smp);
            k<<<grid, kThreads, smp, s>>>(a, nullptr, nullptr, nullptr, nullptr, nullptr, g.fj, g.fi, nullptr);
        }
    } else {
        if (vec) {
            set_smem(stn_out_tile<MODE_DFLOW, true, true>, sm);
            stn_out_tile<MODE_DFLOW, true, true><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                            nullptr, g.fj, g.fi);
        } else {
            set_smem(stn_out_tile<MODE_DFLOW, false, true>, sm);
            stn_out_tile<MODE_DFLOW, false, true><<<grid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, nullptr,
                                                                             nullptr, g.fj, g.fi);
        }
    }
    note_launch();
    return cudaGetLastError();
}

// Side stream + fork/join events for running the d_theta tiles beside the lean d_input
// kernel, once per (host thread, device): no sharing between threads, so concurrent
// calls stay re-entrant; stream-capture safe (the side stream joins a capture through
// the fork event).  Released with the CUDA context.
struct StnFork {
    bool made = false;
    cudaStream_t side;
    cudaEvent_t fork, join;
};
StnFork *stn_fork() {
    static thread_local StnFork f[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    StnFork &x = f[dev];
    if (!x.made) {
        if (cudaStreamCreateWithFlags(&x.side, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
        x.made = true;
    }
    return &x;
}

// Concurrent d_theta tiles and lean d_input when the lean grid is at most this many blocks
// (small batches: both grids end in a partial wave, which the other kernel fills; a
// large batch fills the GPU with either alone -- measured no gain at 64 x 1024^2)
int stn_fork_blocks() {
    const char *e = getenv("RSGRAD_STN_FORK");
    return e ? atoi(e) : 4096;
}

cudaError_t stn_bwd_launch(const StnArgs &a, int algo, int deterministic, void *ws, size_t ws_bytes,
                           cudaStream_t s) {
    (void)ws_bytes;
    const bool det = deterministic && a.dx;
    const StnGeom g = stn_geom(a.H, a.W, a.Ho, a.Wo);
    const StnWs w = stn_ws_layout(ws, a.N, a.C, a.H, a.W, a.Ho, a.Wo, det);
    const long long HW = (long long)a.H * a.W;
    const int tmax = a.Wo > a.Ho ? a.Wo : a.Ho;
    // AUTO / GATHER: cell-owner gather where the preimage is bounded (zeros padding);
    // SCATTER_ATOMIC or border padding: every sample takes the fallback pair.
    const int allow_gather = (algo == 0 || algo == 1) && !a.border && HW * kBCH < (1LL << 31);
    const int variant = stn_bwd_variant();
    const bool vin0 = (a.W % 4 == 0) && aligned16(a.x), vout0 = (a.Wo % 4 == 0) && aligned16(a.dy);
    const long long lean_blocks = (long long)g.bx * ((a.H + kLTY - 1) / kLTY) * a.N;
    if (allow_gather && variant == 2 && !det && vin0 && vout0 && !stn_slow_tiles() && !RS_DTH_LASTBLOCK &&
        lean_blocks <= stn_fork_blocks() && !getenv("RSGRAD_STN_PREP")) {
        // Lean path in three launches: stn_bwd_lean (classifies its sample and computes the
        // normalised coordinates itself), the FAST d_theta tiles (on the side stream for
        // small grids), stn_bwd_tail (d_theta finalize + the fallback samples' scatter)
        const int ly = (a.H + kLTY - 1) / kLTY;
        const dim3 lgrid(g.bx * ly, a.N);
        const int fi_df = (a.Ho + kFIdf - 1) / kFIdf;
        cudaStream_t sdt = s;
        StnFork *fk = nullptr;
        if (a.dx && a.dtheta && (long long)lgrid.x * lgrid.y <= stn_fork_blocks() && (fk = stn_fork()) != nullptr) {
            cudaError_t e = cudaEventRecord(fk->fork, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(fk->side, fk->fork, 0);
            if (e != cudaSuccess) return e;
            sdt = fk->side;
        }
        if (a.dx) {
            const size_t sm = bwd_lean_smem();
            set_smem(stn_bwd_lean<true, true>, sm);
            stn_bwd_lean<true, true><<<lgrid, kThreads, sm, s>>>(a, nullptr, nullptr, nullptr, g.bx, ly,
                                                                 det_ws_layout(w.det, a.N, HW).bar);
            note_launch();
        }
        if (a.dtheta) {
            auto k = stn_out_tile<MODE_DTHETA, true, false, kFIdf, true>;
            const size_t sm = out_tile_smem();
            set_smem(k, sm);
            k<<<dim3(g.fj * fi_df, a.N), kOTFast, sm, sdt>>>(a, nullptr, nullptr, nullptr, w.fb_count, w.pf, g.fj,
                                                              fi_df, nullptr);
            note_launch();
            if (sdt != s) {
                cudaError_t e = cudaEventRecord(fk->join, sdt);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(s, fk->join, 0);
                if (e != cudaSuccess) return e;
            }
        }
        // cooperative (co-resident blocks: the fixed-point scatter's grid barriers)
        int dev = 0;
        cudaGetDevice(&dev);
        static thread_local int cache_nsm[64], cache_occ[64];  // per device, queried once per thread
        const int slot = dev >= 0 && dev < 64 ? dev : 0;
        cudaError_t e = cudaSuccess;
        if (cache_occ[slot] <= 0) {
            cudaDeviceGetAttribute(&cache_nsm[slot], cudaDevAttrMultiProcessorCount, dev);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache_occ[slot], stn_det_tail, kThreads, 0);
            if (e != cudaSuccess) return e;
        }
        const int nsm = cache_nsm[slot], occ = cache_occ[slot];
        if (occ < 1) return cudaErrorInvalidConfiguration;
        StnArgs ta = a;
        const double *pf = w.pf;
        int nf = g.fj * fi_df;
        DetWs dw = det_ws_layout(w.det, a.N, HW);  // one channel plane (cpp = 1)
        void *args[] = {&ta, (void *)&pf, &nf, &dw};
        e = cudaLaunchCooperativeKernel((const void *)stn_det_tail, dim3(nsm * (occ < 2 ? occ : 2)), dim3(kThreads), args,
                                        0, s);
        note_launch();
        return e;
    }
    const DetWs dw = det_ws_layout(w.det, a.N, (det ? (long long)a.C : 1LL) * HW);
    stn_prep_kernel<<<(tmax + 255) / 256, 256, 0, s>>>(a, allow_gather, variant, w.xtab, w.ytab, w.flags, w.fb_list,
                                                       w.fb_count, w.ctr, w.hv_list, w.hv_count, dw.bar);
    note_launch();
    if (!allow_gather && a.dx && !det) {
        cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.C * HW, s);
        if (e != cudaSuccess) return e;
    }
    const bool vin = (a.W % 4 == 0) && aligned16(a.x);
    const bool vout = (a.Wo % 4 == 0) && aligned16(a.dy);
    int tiles_b = g.bx * g.by;
    cudaStream_t sdt = s;  // stream of the d_theta tiles
    StnFork *fk = nullptr;
    if (allow_gather && variant == 2) {
        // lean dX kernel; every sample's d_theta comes from the output-tile kernel
        const size_t sm = bwd_lean_smem();
        const int ly = (a.H + kLTY - 1) / kLTY;
        dim3 grid(g.bx * ly, a.N);
        const bool fast_dth = a.dtheta && (a.W % 4 == 0) && aligned16(a.x) && (a.Wo % 4 == 0) && aligned16(a.dy) &&
                              !stn_slow_tiles();
        if (a.dx && fast_dth && (long long)grid.x * grid.y <= stn_fork_blocks() && (fk = stn_fork()) != nullptr) {
            cudaError_t e = cudaEventRecord(fk->fork, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(fk->side, fk->fork, 0);
            if (e != cudaSuccess) return e;
            sdt = fk->side;
        }
        if (a.dx) {
            if (vout) {
                set_smem(stn_bwd_lean<true>, sm);
                stn_bwd_lean<true><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, g.bx, ly);
            } else {
                set_smem(stn_bwd_lean<false>, sm);
                stn_bwd_lean<false><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, g.bx, ly);
            }
            note_launch();
        }
    } else if (allow_gather && variant == 1) {
        const size_t sm = bwd_gather_smem();
        dim3 grid(g.gx * g.gy, a.N);
        tiles_b = g.gx * g.gy;
        if (vout) {
            set_smem(stn_bwd_gather<true>, sm);
            stn_bwd_gather<true><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, w.pb, g.gx, g.gy);
        } else {
            set_smem(stn_bwd_gather<false>, sm);
            stn_bwd_gather<false><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, w.pb, g.gx, g.gy);
        }
        note_launch();
    } else if (allow_gather) {
        const size_t sm = bwd_cell_smem();
        dim3 grid(g.bx * g.by, a.N);
        if (vout) {
            set_smem(stn_bwd_cell<true>, sm);
            stn_bwd_cell<true><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, w.pb, g.bx, g.by);
        } else {
            set_smem(stn_bwd_cell<false>, sm);
            stn_bwd_cell<false><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, w.flags, w.pb, g.bx, g.by);
        }
        note_launch();
    }
    // fallback samples (all samples when !allow_gather or the lean dX kernel):
    // d_theta from output tiles ...
    const bool dth_all = allow_gather && variant == 2;
    const bool dth_fast = vin && vout && dth_all && !stn_slow_tiles();
    const int fi_df = (a.Ho + kFIdf - 1) / kFIdf;  // d_theta tiles per column, fast path
    // fallback d_input: per-tap global atomics (AUTO, SCATTER_ATOMIC), or block-private
    // footprint accumulation (SCATTER_PRIV; measured slower on sm_100, where shared-memory
    // float atomics are CAS loops: 3.45 vs 3.10 ms at 16x16x1024^2)
    const bool priv = a.dx && algo == 2;
    const size_t sm = out_tile_smem(), smp = sm + sizeof(float) * kFStage;
    if (a.dtheta) {
        dim3 grid(g.fj * g.fi, dth_all ? a.N : 1);
        const int *fbl = dth_all ? nullptr : w.fb_list;
        if (dth_fast) {
            auto k = stn_out_tile<MODE_DTHETA, true, false, kFIdf, true>;
            set_smem(k, sm);
            grid.x = g.fj * fi_df;
            k<<<grid, kOTFast, sm, sdt>>>(a, w.xtab, w.ytab, nullptr, w.fb_count, w.pf, g.fj, fi_df,
                                          RS_DTH_LASTBLOCK ? w.ctr : nullptr);
            if (sdt != s) {  // join: the finalize (and the caller) see the tiles' partials
                cudaError_t e = cudaEventRecord(fk->join, sdt);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(s, fk->join, 0);
                if (e != cudaSuccess) return e;
            }
        } else if (priv && !dth_all) {  // fallback samples: d_theta and privatised d_input
            auto k = vin ? stn_out_tile<MODE_DTHETA, true, false, kFIdth, false, true>
                         : stn_out_tile<MODE_DTHETA, false, false, kFIdth, false, true>;
            set_smem(k, smp);
            k<<<grid, kThreads, smp, s>>>(a, w.xtab, w.ytab, fbl, w.fb_count, w.pf, g.fj, g.fi, nullptr);
        } else if (vin) {
            set_smem(stn_out_tile<MODE_DTHETA, true>, sm);
            stn_out_tile<MODE_DTHETA, true><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, fbl, w.fb_count,
                                                                       w.pf, g.fj, g.fi);
        } else {
            set_smem(stn_out_tile<MODE_DTHETA, false>, sm);
            stn_out_tile<MODE_DTHETA, false><<<grid, kThreads, sm, s>>>(a, w.xtab, w.ytab, fbl, w.fb_count,
                                                                        w.pf, g.fj, g.fi);
        }
        note_launch();
    }
    if (a.dx && priv && (dth_all || !a.dtheta)) {
        // fallback samples' d_input alone: MODE_DFLOW with affine coordinates, no d_flow
        StnArgs b = a;
        b.dflow = nullptr;
        auto k = vin ? stn_out_tile<MODE_DFLOW, true, false, kFIdth, false, true>
                     : stn_out_tile<MODE_DFLOW, false, false, kFIdth, false, true>;
        set_smem(k, smp);
        k<<<dim3(g.fj * g.fi, 1), kThreads, smp, s>>>(b, w.xtab, w.ytab, w.fb_list, w.fb_count, nullptr, g.fj, g.fi, nullptr);
        note_launch();
    } else if (det) {
        // deterministic=1: the fallback samples' d_input by the fixed-point scatter
        const StnTapSampler smp{a.theta, a.H, a.W, a.Ho, a.Wo, a.ac, a.border};
        cudaError_t e = det_scatter_launch(smp, a.dy, a.dx, a.N, a.C, HW, (long long)a.Ho * a.Wo, w.fb_list,
                                           w.fb_count, nullptr, w.det, s);
        if (e != cudaSuccess) return e;
    } else if (a.dx && !priv) {
        const long long P = (long long)a.Ho * a.Wo;
        // grid-stride over the fallback list: when every sample is a fallback (border
        // padding, SCATTER_ATOMIC) a full grid; else (usually empty) a small one that exits at once
        long long blocks = (P + kThreads - 1) / kThreads;
        const long long cap = allow_gather ? 2 * kNumSMs : 4 * kNumSMs * 8;
        if (blocks > cap) blocks = cap;
        stn_dx_scatter<<<(unsigned)blocks, kThreads, 0, s>>>(a, w.fb_list, w.fb_count);
        note_launch();
        // heavy fallback samples (skipped by the atomic scatter): the exact fixed-point scatter
        const StnTapSampler hsmp{a.theta, a.H, a.W, a.Ho, a.Wo, a.ac, a.border};
        cudaError_t e = det_scatter_launch(hsmp, a.dy, a.dx, a.N, a.C, HW, P, w.hv_list, w.hv_count, nullptr, w.det, s,
                                           1, false, 1, 1);
        if (e != cudaSuccess) return e;
    }
    if (a.dtheta && !(dth_fast && RS_DTH_LASTBLOCK)) {  // (else the FAST tiles finalize in their last block)
        stn_dtheta_finalize<<<a.N, kThreads, 0, s>>>(w.pb, tiles_b, w.pf, g.fj * (dth_fast ? fi_df : g.fi),
                                                      dth_all ? nullptr : w.flags, a.dtheta);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace rs
