// det.cuh — deterministic general scatter by fixed-point integer accumulation.
//
// where a scatter cannot be converted to a gather, "we fall back to a
// general scattering operation" with atomics.  fp32 atomics sum in the order the
// memory system applies them, so their result is not reproducible (and their rounding
// grows with the fan-in of an element).  This path makes the same scatter bitwise
// reproducible (rs_opts.deterministic = 1, SURVEY §8(b) "Deterministic when
// deterministic=1"): every contribution w*g is formed exactly in fp64, scaled by 2^S
// and rounded once to a 64-bit integer, and the integers are summed with 64-bit
// atomics -- integer addition is associative, so the sum does not depend on the
// order.  S is chosen per sample from max|dY| so that no partial sum can overflow:
//   |sum| <= max|g| * sum_q |w_q| <= max|g| * P * kWmax  < 2^61 * 2^-S.
// Each term carries at most 2^-(S+1) absolute rounding, so an element with n terms
// is within n * 2^-(S+1) = n * max|g| * P * kWmax * 2^-62 of the exact sum (≈1e-11
// for the bench shapes) -- far tighter than fp32 accumulation.
//
// One persistent cooperative kernel walks the selected samples one after another
// (the int64 accumulator is one sample large): per sample, (A) zero the accumulator
// and reduce max|dY| (order-free: atomicMax on the bit pattern), (B) scatter, (C)
// convert to fp32 into dx; phases are separated by a grid barrier (all blocks are
// co-resident: cudaLaunchCooperativeKernel).
#pragma once

#include "common.cuh"

namespace rs {

struct DetWs {
    unsigned long long *acc;  // C*HW accumulators of one sample
    unsigned *maxbits;        // per selected-sample slot: max |dY| bit pattern
    unsigned *bar;            // grid barrier: count, generation
};

inline size_t det_align(size_t v) { return (v + 255) & ~(size_t)255; }

// bytes of the deterministic-scatter workspace for N samples of C*HW input elements
inline size_t det_ws_bytes(int N, long long CHW) {
    return det_align(sizeof(unsigned long long) * (size_t)CHW) + det_align(sizeof(unsigned) * ((size_t)N + 2));
}

inline DetWs det_ws_layout(void *base, int N, long long CHW) {
    (void)N;
    DetWs w;
    char *b = (char *)base;
    w.acc = (unsigned long long *)b;
    w.bar = (unsigned *)(b + det_align(sizeof(unsigned long long) * (size_t)CHW));
    w.maxbits = w.bar + 2;
    return w;
}

// Sense-free grid barrier: the generation is read before arriving; the last block
// to arrive resets the count and bumps the generation.
RS_DEV void det_grid_barrier(unsigned *bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(100);
        }
        __threadfence();
    }
    __syncthreads();
}

// Sampler concept (see the layer files):
//   static constexpr int kMaxTaps;      taps per output pixel
//   static constexpr double kWmax;      bound on sum over output pixels of |w| landing on one element, / P
//   RS_DEV int taps(int n, long long q, long long *off, float *w) const;
//     the in-image taps of output pixel q of sample n: element offsets within a
//     channel plane and the fp32 weights the float path uses.
// Sample selection: list/count (device list of samples), else flags (flags[n] != 0),
// else every sample 0..N-1.  flags[n] == flag_on selects (a per-call tag lets a flag array
// be reused without clearing it: stale values only cost a recompute, never correctness).
// One sample's exact scatter, by every block of a co-resident grid (three phases
// separated by grid barriers; max-slot `slot` of ws.maxbits must be zero on entry).
// cpp > 0: the accumulator holds cpp channel planes and the channels are walked in groups
// of cpp (zero / scatter / convert per group: a small workspace for rare samples).
template <class S, int kT>
RS_DEV void det_scatter_one(const S &smp, const float *__restrict__ dy, float *__restrict__ dx, int n, int slot, int C,
                            long long HW, long long P, const DetWs &ws, unsigned *red, int cpp = 0) {
    const unsigned nb = gridDim.x;
    const long long tid = (long long)blockIdx.x * kT + threadIdx.x, nthr = (long long)nb * kT;
    const long long CP = (long long)C * P;
    const float *g = dy + (long long)n * CP;
    if (cpp <= 0 || cpp > C) cpp = C;
    // max |dY| of the sample
    unsigned m = 0u;
    for (long long e = tid; e < CP; e += nthr) m = max(m, __float_as_uint(fabsf(__ldg(g + e))));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned b = 0u;
        for (int k = 0; k < kT / 32; k++) b = max(b, red[k]);
        atomicMax(ws.maxbits + slot, b);
    }
    det_grid_barrier(ws.bar, nb);
    const float mx = __uint_as_float(__ldcg(ws.maxbits + slot));
    const bool finite = isfinite(mx);
    int Sx = 0;
    if (mx > 0.f && finite) {
        const double bound = (double)mx * (double)P * S::kWmax;
        Sx = 61 - ilogb(bound) - 1;  // bound < 2^(ilogb+1)  =>  bound * 2^S < 2^61
    }
    for (int c0 = 0; c0 < C; c0 += cpp) {
        const int cn = min(cpp, C - c0);
        const long long GHW = (long long)cn * HW;
        // (A) zero the accumulator of this channel group
        for (long long e = tid; e < GHW; e += nthr) ws.acc[e] = 0ull;
        det_grid_barrier(ws.bar, nb);
        // (B) scatter: round(w*g * 2^S) into 64-bit integer sums
        if (finite) {
            for (long long q = tid; q < P; q += nthr) {
                long long off[S::kMaxTaps];
                float w[S::kMaxTaps];
                const int nt = smp.taps(n, q, off, w);
                if (nt == 0) continue;
                for (int c = 0; c < cn; c++) {
                    const float gv = __ldg(g + (long long)(c0 + c) * P + q);
                    if (gv == 0.f) continue;
                    unsigned long long *ac = ws.acc + (long long)c * HW;
#pragma unroll
                    for (int k = 0; k < S::kMaxTaps; k++) {
                        if (k >= nt) break;
                        const double v = ldexp((double)w[k] * (double)gv, Sx);  // exact product, exact scaling
                        const long long iv = __double2ll_rn(v);
                        if (iv != 0) atomicAdd(ac + off[k], (unsigned long long)iv);
                    }
                }
            }
        }
        det_grid_barrier(ws.bar, nb);
        // (C) fixed point -> fp32 (non-finite dY: the sample's dx is NaN)
        float *d = dx + ((long long)n * C + c0) * HW;
        for (long long e = tid; e < GHW; e += nthr)
            d[e] = finite ? (float)ldexp((double)(long long)__ldcg(ws.acc + e), -Sx) : __int_as_float(0x7fffffff);
        det_grid_barrier(ws.bar, nb);
    }
}

template <class S, int kT = 256>
__global__ void __launch_bounds__(kT)
    det_scatter_kernel(S smp, const float *__restrict__ dy, float *__restrict__ dx, int N, int C, long long HW,
                       long long P, const int *__restrict__ list, const int *__restrict__ count,
                       int *__restrict__ flags, int flag_on, DetWs ws, int cpp = 0) {
    const int nsel = list ? *count : N;
    __shared__ unsigned red[kT / 32];
    if (!list && flags) {
        // flag-selected samples (the AUTO warp rescue, usually none): one parallel pass over
        // the flags first, so a call without a selected sample exits after one load
        // latency instead of N dependent ones
        int any = 0;
        for (int n = threadIdx.x; n < N; n += kT) any |= flags[n] == flag_on;
        if (!__syncthreads_or(any)) return;
    }
    for (int f = 0; f < nsel; f++) {
        const int n = list ? list[f] : f;
        if (!list && flags && flags[n] != flag_on) continue;  // uniform over the grid
        det_scatter_one<S, kT>(smp, dy, dx, n, f, C, HW, P, ws, red, cpp);
        // every block has read flags[n]: clear it, so a CUDA-graph replay (same tag) does
        // not recompute the sample again unless it is flagged anew
        if (flags && !list && (long long)blockIdx.x * kT + threadIdx.x == 0) flags[n] = 0;
    }
}
// Zero the barrier / max slots, then launch the cooperative kernel with every block
// co-resident.
template <class S>
cudaError_t det_scatter_launch(const S &smp, const float *dy, float *dx, int N, int C, long long HW, long long P,
                               const int *list, const int *count, int *flags, void *ws, cudaStream_t s,
                               int flag_on = 1, bool zero_slots = true, int max_blocks_per_sm = 4, int cpp = 0) {
    constexpr int kT = 256;
    const DetWs w = det_ws_layout(ws, N, (long long)(cpp > 0 && cpp < C ? cpp : C) * HW);
    cudaError_t e = cudaSuccess;
    if (zero_slots) {  // (else the caller's previous kernel on s zeroed them)
        e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned) * ((size_t)N + 2), s);
        if (e != cudaSuccess) return e;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = det_scatter_kernel<S, kT>;
    // SM count and occupancy per (kernel instantiation, device), queried once per thread
    static thread_local int cache_nsm[64], cache_occ[64];
    const int slot = dev >= 0 && dev < 64 ? dev : 0;
    if (cache_occ[slot] <= 0) {
        cudaDeviceGetAttribute(&cache_nsm[slot], cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache_occ[slot], kern, kT, 0);
        if (e != cudaSuccess) return e;
    }
    const int nsm = cache_nsm[slot], occ = cache_occ[slot];
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int blocks = nsm * (occ < max_blocks_per_sm ? occ : max_blocks_per_sm);
    S sm = smp;
    long long hw = HW, p = P;
    int n = N, c = C, fo = flag_on, cp = cpp;
    DetWs wk = w;
    void *args[] = {&sm, (void *)&dy, (void *)&dx, &n, &c, &hw, &p, (void *)&list, (void *)&count, (void *)&flags, &fo,
                    &wk, &cp};
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(blocks), dim3(kT), args, 0, s);
    note_launch();
    return e;
}

}  // namespace rs
