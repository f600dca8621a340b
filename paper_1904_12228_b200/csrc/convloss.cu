// convloss.cu — the checkpointing study of PAPER.md:795-828 and the input(x/4)
// upsampling adjoint of PAPER.md:725-731, sm_100a.
//
// d_in of loss = sum (conv(in, k) - target)^2 is "a cross correlation of
// 2*(convolved-target) with kernel".  With the residual
//   R(v) = 2 (sum_r in(v - r + p) k(r) - target(v))   (zero outside the image)
// it is d_in(u) = sum_r k(r) R(u + r - p), p = (kh/2, kw/2) (R11).
// The three schedules the paper times:
//   compute_root    cl_residual writes R to memory, cl_gather reads it back;
//   compute_inline  cl_inline recomputes R at every tap (kh*kw * kh*kw MACs per px);
//   compute_at      cl_tiled computes R for a 32 x 32 tile of d_in (+ halo) in shared
//                   memory from a staged input window, then gathers from it.
// upsample4_fwd/bwd: y(x) = in(x/4) and its converted gather d_in(x) = sum_r d_out(4x + r).
#include "common.cuh"

namespace rs {
namespace {

constexpr int kLT = 256;
constexpr int kTS = 32;  // compute_at tile (d_in), threads 32 x 8, 4 rows each

struct KW49 {
    float w[49];
};

RS_DEV float in_at(const float *p, int H, int W, int y, int x) {
    return (y >= 0 && y < H && x >= 0 && x < W) ? __ldg(p + (long long)y * W + x) : 0.f;
}

// residual at v (inside the image)
RS_DEV float residual(const float *in, const float *tg, int H, int W, int kh, int kw, const KW49 &k, int vy,
                      int vx) {
    const int py = kh / 2, px = kw / 2;
    float c = 0.f;
    for (int ry = 0; ry < kh; ry++)
        for (int rx = 0; rx < kw; rx++) c = fmaf(in_at(in, H, W, vy - ry + py, vx - rx + px), k.w[ry * kw + rx], c);
    return 2.f * (c - __ldg(tg + (long long)vy * W + vx));
}

__global__ void __launch_bounds__(kLT)
    cl_residual(const float *in, const float *tg, float *R, int H, int W, int kh, int kw, KW49 k) {
    const long long HW = (long long)H * W;
    const int n = blockIdx.y;
    const int i = blockIdx.x * kLT + threadIdx.x;
    if (i >= HW) return;
    const int y = i / W, x = i - y * W;
    R[n * HW + i] = residual(in + n * HW, tg + n * HW, H, W, kh, kw, k, y, x);
}

__global__ void __launch_bounds__(kLT)
    cl_gather(const float *R, float *din, int H, int W, int kh, int kw, KW49 k) {
    const long long HW = (long long)H * W;
    const int n = blockIdx.y;
    const int i = blockIdx.x * kLT + threadIdx.x;
    if (i >= HW) return;
    const int y = i / W, x = i - y * W;
    const int py = kh / 2, px = kw / 2;
    const float *Rn = R + n * HW;
    float d = 0.f;
    for (int ry = 0; ry < kh; ry++)
        for (int rx = 0; rx < kw; rx++) d = fmaf(k.w[ry * kw + rx], in_at(Rn, H, W, y + ry - py, x + rx - px), d);
    din[n * HW + i] = d;
}

__global__ void __launch_bounds__(kLT)
    cl_inline(const float *in, const float *tg, float *din, int H, int W, int kh, int kw, KW49 k) {
    const long long HW = (long long)H * W;
    const int n = blockIdx.y;
    const int i = blockIdx.x * kLT + threadIdx.x;
    if (i >= HW) return;
    const int y = i / W, x = i - y * W;
    const int py = kh / 2, px = kw / 2;
    float d = 0.f;
    for (int ry = 0; ry < kh; ry++)
        for (int rx = 0; rx < kw; rx++) {
            const int vy = y + ry - py, vx = x + rx - px;
            if (vy < 0 || vy >= H || vx < 0 || vx >= W) continue;
            d = fmaf(k.w[ry * kw + rx], residual(in + n * HW, tg + n * HW, H, W, kh, kw, k, vy, vx), d);
        }
    din[n * HW + i] = d;
}

// compute_at: per 32 x 32 tile of d_in, R on the tile + (kh-1, kw-1) halo in shared
// memory, computed from the input window with a second halo.
__global__ void __launch_bounds__(kLT)
    cl_tiled(const float *in, const float *tg, float *din, int H, int W, int kh, int kw, KW49 k, int tiles_x) {
    extern __shared__ float cls[];
    const int py = kh / 2, px = kw / 2;
    const int RH = kTS + kh - 1, RW = kTS + kw - 1;
    const int IH = kTS + 2 * (kh - 1), IW = kTS + 2 * (kw - 1);
    float *sI = cls;            // IH x IW
    float *sR = cls + IH * IW;  // RH x RW
    const long long HW = (long long)H * W;
    const int n = blockIdx.y;
    const int x0 = (blockIdx.x % tiles_x) * kTS, y0 = (blockIdx.x / tiles_x) * kTS;
    const float *inn = in + n * HW, *tgn = tg + n * HW;
    // R rows v_y in [y0 - py, y0 + kTS - 1 + kh - 1 - py]; input rows in [y0 - (kh-1), ...]
    const int ry0 = y0 - py, rx0 = x0 - px;
    const int iy0 = y0 - (kh - 1), ix0 = x0 - (kw - 1);
    for (int e = threadIdx.x; e < IH * IW; e += kLT) {
        const int r = e / IW, c = e - r * IW;
        sI[e] = in_at(inn, H, W, iy0 + r, ix0 + c);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RH * RW; e += kLT) {
        const int r = e / RW, c = e - r * RW;
        const int vy = ry0 + r, vx = rx0 + c;
        float v = 0.f;
        if (vy >= 0 && vy < H && vx >= 0 && vx < W) {
            // in(vy - ry + py) sits at window row vy - ry + py - iy0 = r + (kh-1) - ry
            float cacc = 0.f;
            for (int ry = 0; ry < kh; ry++)
                for (int rx = 0; rx < kw; rx++)
                    cacc = fmaf(sI[(r + kh - 1 - ry) * IW + c + kw - 1 - rx], k.w[ry * kw + rx], cacc);
            v = 2.f * (cacc - __ldg(tgn + (long long)vy * W + vx));
        }
        sR[e] = v;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int h = 0; h < kTS / 8; h++) {
        const int yl = ty + 8 * h, y = y0 + yl, x = x0 + tx;
        if (y >= H || x >= W) continue;
        // R(y + ry - py) sits at R row yl + ry
        float d = 0.f;
        for (int ry = 0; ry < kh; ry++)
            for (int rx = 0; rx < kw; rx++) d = fmaf(k.w[ry * kw + rx], sR[(yl + ry) * RW + tx + rx], d);
        din[n * HW + (long long)y * W + x] = d;
    }
}

// thread per input element: writes its 4 x 4 output block (4 float4 rows when aligned)
__global__ void __launch_bounds__(kLT) up4_fwd(const float *x, float *y, long long total, int W, bool vec) {
    const long long i = (long long)blockIdx.x * kLT + threadIdx.x;
    if (i >= total) return;
    const long long row = i / W;  // (n, c, yy) flattened
    const int xx = (int)(i - row * W);
    const float v = __ldg(x + i);
    float *o = y + (row * 4) * (4LL * W) + 4LL * xx;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        if (vec) {
            *(float4 *)(o + r * 4LL * W) = make_float4(v, v, v, v);
        } else {
#pragma unroll
            for (int c = 0; c < 4; c++) o[r * 4LL * W + c] = v;
        }
    }
}

// the converted gather: d_in(x) = sum_{r < 4 x 4} d_out(4x + r)
__global__ void __launch_bounds__(kLT) up4_bwd(const float *dy, float *dx, long long total, int W, bool vec) {
    const long long i = (long long)blockIdx.x * kLT + threadIdx.x;
    if (i >= total) return;
    const long long row = i / W;
    const int xx = (int)(i - row * W);
    const float *g = dy + (row * 4) * (4LL * W) + 4LL * xx;
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        float4 v;
        if (vec) {
            v = __ldg((const float4 *)(g + r * 4LL * W));
        } else {
            const float *q = g + r * 4LL * W;
            v = make_float4(__ldg(q), __ldg(q + 1), __ldg(q + 2), __ldg(q + 3));
        }
        s += (v.x + v.y) + (v.z + v.w);
    }
    dx[i] = s;
}

KW49 pack_k(const float *hk, int n) {
    KW49 k{};
    for (int i = 0; i < n && i < 49; i++) k.w[i] = hk[i];
    return k;
}

}  // namespace

size_t convloss_ws_bytes(int N, int H, int W) { return sizeof(float) * (size_t)N * H * W; }

cudaError_t convloss_grad_launch(const float *in, const float *hk, const float *tg, int N, int H, int W, int kh,
                                 int kw, int schedule, float *din, void *ws, cudaStream_t s) {
    const KW49 k = pack_k(hk, kh * kw);
    const long long HW = (long long)H * W;
    const dim3 g1((unsigned)((HW + kLT - 1) / kLT), N);
    if (schedule == 0) {
        float *R = (float *)ws;
        cl_residual<<<g1, kLT, 0, s>>>(in, tg, R, H, W, kh, kw, k);
        note_launch();
        cl_gather<<<g1, kLT, 0, s>>>(R, din, H, W, kh, kw, k);
        note_launch();
    } else if (schedule == 1) {
        cl_inline<<<g1, kLT, 0, s>>>(in, tg, din, H, W, kh, kw, k);
        note_launch();
    } else {
        const int tiles_x = (W + kTS - 1) / kTS, tiles_y = (H + kTS - 1) / kTS;
        const size_t sm = sizeof(float) * ((size_t)(kTS + 2 * (kh - 1)) * (kTS + 2 * (kw - 1)) +
                                           (size_t)(kTS + kh - 1) * (kTS + kw - 1));
        cl_tiled<<<dim3(tiles_x * tiles_y, N), kLT, sm, s>>>(in, tg, din, H, W, kh, kw, k, tiles_x);
        note_launch();
    }
    return cudaGetLastError();
}

cudaError_t upsample4_launch(const float *src, float *dst, int N, int C, int H, int W, bool bwd, cudaStream_t s) {
    const long long total = (long long)N * C * H * W;
    const unsigned blocks = (unsigned)((total + kLT - 1) / kLT);
    const float *big = bwd ? src : dst;  // the 4H x 4W side: 16-B rows when aligned
    const bool vec = (((uintptr_t)big) & 15u) == 0;
    if (bwd) up4_bwd<<<blocks, kLT, 0, s>>>(src, dst, total, W, vec);
    else up4_fwd<<<blocks, kLT, 0, s>>>(src, dst, total, W, vec);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rs
