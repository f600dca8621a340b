// common.cuh — device helpers shared by the rsgrad kernels (product path only).
//
// Precision contract (P1): every SAMPLE COORDINATE is evaluated in
// fp64 with explicit round-to-nearest intrinsics (__dadd_rn/__dmul_rn/
// __ddiv_rn) in the left-to-right order of the definition, so no FMA
// contraction can move a coordinate across an integer: the cell a sample lands
// in is the exact fp64 cell of the definition.  Fractions are then rounded to
// fp32 and all data arithmetic (weights, taps, sums) is fp32.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define RS_DEV __device__ __forceinline__

namespace rs {

constexpr int kNumSMs = 148;  // B200

// ----------------------------------------------------------------- launch accounting
void note_launch();  // api.cu: thread-local counter behind rsgrad_launch_count()

// ----------------------------------------------------------------- STN coordinates (R1)
// normalised output coordinate of index j on an axis of length L
RS_DEV double stn_norm(int j, int L, int ac) {
    if (ac) return __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, (double)j), (double)(L - 1)));
    return __dsub_rn(__ddiv_rn(__dadd_rn(__dmul_rn(2.0, (double)j), 1.0), (double)L), 1.0);
}

// un-normalise a grid coordinate g to pixel units on an axis of length L
RS_DEV double stn_unnorm(double g, int L, int ac) {
    if (ac) return __dmul_rn(__dmul_rn(__dadd_rn(g, 1.0), (double)(L - 1)), 0.5);
    return __dmul_rn(__dsub_rn(__dmul_rn(__dadd_rn(g, 1.0), (double)L), 1.0), 0.5);
}

// g = t0*a + t1*b + t2, evaluated as ((t0*a) + (t1*b)) + t2
RS_DEV double affine3(double t0, double t1, double t2, double a, double b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(t0, a), __dmul_rn(t1, b)), t2);
}

// Border padding: clamp to [0, L-1]; derivative 1 strictly inside, else 0.
RS_DEV double clamp_coord(double v, int L, float &dclamp) {
    if (v <= 0.0) { dclamp = 0.f; return 0.0; }
    if (v >= (double)(L - 1)) { dclamp = 0.f; return (double)(L - 1); }
    dclamp = 1.f;
    return v;
}

// Floor cell of a coordinate: integer corner and fp32 fraction.
struct Cell {
    int i0;
    float f;
};
RS_DEV Cell cell_of(double v) {
    double fl = floor(v);
    Cell c;
    // coordinates beyond +-2^30 px are far outside any image: clamp the
    // integer so the bounds tests below stay well defined (weights unchanged)
    c.i0 = fl < -1073741824.0 ? -1073741824 : (fl > 1073741824.0 ? 1073741824 : (int)fl);
    c.f = (float)__dsub_rn(v, fl);
    return c;
}

// ----------------------------------------------------------------- cheap integer division
// a / d for 0 <= a < 2^31, d >= 1, via a double reciprocal and a one-step fix-up
// (avoids the 64-bit software division routine in per-pixel index math).
RS_DEV int fast_div(int a, int d, double inv_d) {
    int q = (int)((double)a * inv_d);
    if (q * d > a) q--;
    if ((q + 1) * d <= a) q++;
    return q;
}

// ----------------------------------------------------------------- reductions
RS_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

RS_DEV double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Vector reduction to global memory without return (sm_90+): 4 consecutive floats.
RS_DEV void red_add_v4(float *addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
}

RS_DEV void red_add(float *addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

// streaming loads / stores (read-once data: no L1 allocation)
RS_DEV float ldg_stream(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// read-only gather load with a 128-B L2 fetch hint (the neighbours of a bilinear tap
// are read by adjacent lanes / rows soon after)
RS_DEV float ldg_tap(const float *p) {
    float v;
    asm volatile("ld.global.nc.L2::128B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

RS_DEV float4 ldg_stream4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

RS_DEV void stg_stream(float *p, float v) {
    asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ----------------------------------------------------------------- cp.async (LDGSTS) staging
RS_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
RS_DEV void cp_async16(void *s, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
// zero-filling variants: ok = false copies 0 source bytes (the 16 / 4 B are zeroed)
RS_DEV void cp_async16_zfill(void *s, const void *g, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(ok ? 16 : 0)
                 : "memory");
}
RS_DEV void cp_async4_zfill(void *s, const void *g, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(ok ? 4 : 0)
                 : "memory");
}
RS_DEV void cp_async4(void *s, const void *g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
RS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
RS_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ----------------------------------------------------------------- mbarrier (cp.async completion)
RS_DEV void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
RS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// arrive on `bar` once all of this thread's earlier cp.async copies have landed
// (.noinc: the arrival counts against the count the barrier was initialised with)
RS_DEV void cp_async_arrive(unsigned long long *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RS_DEV void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RS_DEV bool mbar_try_wait(unsigned long long *bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the thread sleeps until the phase completes (or
// the hint expires) instead of spinning through issue slots
RS_DEV bool mbar_try_wait_sleep(unsigned long long *bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}
RS_DEV void mbar_wait(unsigned long long *bar, unsigned parity) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
}
// 16-B cp.async to a shared-window address (no generic->shared conversion per copy)
RS_DEV void cp_async16_s(unsigned s, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}

// Compact row layout of a staged footprint: row r holds columns [xa[r], xa[r]+cnt[r])
// of source row (ybase + r) at smem offset off[r] (16-B aligned when VEC).
// Built by warp 0 from inclusive column ranges [lo[r], hi[r]] (lo > hi: empty row).
template <bool VEC>
RS_DEV void build_rows(int R, int Wlim, const int *lo, const int *hi, int *xa, int *off, int *cnt,
                       int *Fout) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    int run = 0;
    for (int base = 0; base < R; base += 32) {
        const int r = base + lane;
        int width = 0, a0 = 0, n = 0;
        if (r < R && lo[r] <= hi[r]) {
            a0 = VEC ? (lo[r] & ~3) : lo[r];
            const int e = VEC ? min(Wlim, (hi[r] + 4) & ~3) : hi[r] + 1;
            n = e - a0;
            width = (n + 3) & ~3;
        }
        int v = width;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (r < R) {
            xa[r] = a0;
            cnt[r] = n;
            off[r] = run + v - width;
        }
        run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) *Fout = run;
}

// sum of cnt[0..R) (floats actually copied per channel), by warp 0
RS_DEV void sum_rows(int R, const int *cnt, int *out) {
    if (threadIdx.x >= 32) return;
    int s = 0;
    for (int r = threadIdx.x; r < R; r += 32) s += cnt[r];
    s = __reduce_add_sync(0xffffffffu, s);
    if (threadIdx.x == 0) *out = s;
}

// Issue cp.async copies of nch channel planes' rows (channel stride cstride floats)
// into dst + c*F + off[r].  Eight lanes per row (4 rows per warp instruction), the
// channel loop innermost; no integer division.
template <bool VEC>
RS_DEV void stage_rows(float *dst, int F, const float *base, long long cstride, int nch, int R,
                       int W, int ybase, const int *xa, const int *off, const int *cnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sub = lane >> 3, l8 = lane & 7;
    for (int r = warp * 4 + sub; r < R; r += nw * 4) {
        const int w = cnt[r];
        const float *src = base + (long long)(ybase + r) * W + xa[r];
        float *d = dst + off[r];
        for (int c = 0; c < nch; c++) {
            if (VEC) {
                for (int q = l8 * 4; q < w; q += 32) cp_async16(d + q, src + q);
            } else {
                for (int q = l8; q < w; q += 8) cp_async4(d + q, src + q);
            }
            src += cstride;
            d += F;
        }
    }
}
}  // namespace rs

// ----------------------------------------------------------------- launchers (internal ABI)
namespace rs {
struct StnArgs {
    const float *x, *theta, *dy;
    float *y, *dx, *dtheta;
    int N, C, H, W, Ho, Wo;
    int ac, border;
    const float *flow;  // warp layer through the output-tile kernel (theta unused)
    float *dflow;
};
struct WarpArgs {
    const float *x, *flow, *dy;
    float *y, *dx, *dflow;
    int N, C, H, W;
    int border;
};
struct BsliceArgs {
    const float *grid, *guide, *x, *dy;
    float *y, *dgrid, *dguide, *dx;
    int N, H, W, D, Gh, Gw;
};

struct ConvArgs {
    const float *x, *k, *dy;
    float *y, *dx, *dk;
    int N, Ci, Co, H, W, kh, kw;
};

// each returns a cudaError_t from the launches; algo is an rs_algo value
cudaError_t stn_fwd_launch(const StnArgs &a, cudaStream_t s);
cudaError_t stn_bwd_launch(const StnArgs &a, int algo, int deterministic, void *ws, size_t ws_bytes,
                           cudaStream_t s);
size_t stn_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det = false);

// output-tile kernel driven by a flow field (warp.cu): mode 0 = y, 2 = d_flow (+ dx reds)
cudaError_t flow_tile_launch(const StnArgs &a, int mode, bool priv, cudaStream_t s);
cudaError_t warp_fwd_launch(const WarpArgs &a, cudaStream_t s);
cudaError_t warp_bwd_launch(const WarpArgs &a, int algo, int deterministic, void *ws,
                            size_t ws_bytes, cudaStream_t s);
size_t warp_ws_bytes(int N, int C, int H, int W, bool det = false);

cudaError_t bslice_fwd_launch(const BsliceArgs &a, cudaStream_t s);
cudaError_t bslice_bwd_launch(const BsliceArgs &a, int algo, int deterministic, void *ws,
                              size_t ws_bytes, cudaStream_t s);
size_t bslice_ws_bytes(int N, int H, int W, int D, int Gh, int Gw);
size_t bslice_det_ws_bytes(int N, int D, int Gh, int Gw);
size_t bslice_bwd_ws_bytes(int N, int H, int W, int D, int Gh, int Gw, bool det);

bool conv_shape_ok(int Ci, int Co, int kh, int kw);
cudaError_t conv_fwd_launch(const ConvArgs &a, cudaStream_t s);
cudaError_t conv_bwd_launch(const ConvArgs &a, int algo, void *ws, size_t ws_bytes, cudaStream_t s);
size_t conv_ws_bytes(int N, int Ci, int Co, int H, int W, int kh, int kw);

size_t convloss_ws_bytes(int N, int H, int W);
cudaError_t convloss_grad_launch(const float *in, const float *hk, const float *tg, int N, int H, int W, int kh,
                                 int kw, int schedule, float *din, void *ws, cudaStream_t s);
cudaError_t upsample4_launch(const float *src, float *dst, int N, int C, int H, int W, bool bwd, cudaStream_t s);

size_t stn_var_ws_bytes(int N, int P, int ne);
size_t stn_bicubic_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det);
cudaError_t stn_bicubic_launch(const StnArgs &a, bool bwd, int algo, bool det, void *ws, cudaStream_t s);
cudaError_t stn_lanczos_launch(const StnArgs &a, bool bwd, bool det, void *ws, cudaStream_t s);
cudaError_t stn3d_launch(const float *x, const float *theta, const float *dy, float *y, float *dx, float *dtheta,
                         int N, int C, int D, int H, int W, int Do, int Ho, int Wo, int ac, bool bwd, bool det,
                         void *ws, cudaStream_t s);
size_t stn_lanczos_ws_bytes(int N, int C, int H, int W, int Ho, int Wo, bool det);
size_t stn3d_ws_bytes(int N, int C, int D, int H, int W, int Do, int Ho, int Wo, bool det);
}  // namespace rs
