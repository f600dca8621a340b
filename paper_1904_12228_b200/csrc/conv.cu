// conv.cu — 2-D convolution layer and its adjoint, sm_100a.
//
// The paper's only quantified scatter-vs-gather comparison is "the backward pass of
// a 2D convolution layer applied to a 16 x 16 x 256 x 256 input takes 68 ms using
// atomics and 6 ms with our scatter-to-gather conversion".  The
// layer is the paper's gather output(x) = input(x - r.x) * kernel(r.x)
// in 2-D with channels, centred (R10):
//   y[n,co,y,x] = sum_{ci,ry,rx} x[n,ci, y-ry+ph, x-rx+pw] k[co,ci,ry,rx].
//
// Kernels
//   conv_direct      out[n,o,y,x] = sum_{i,ry,rx} in[n,i, y+s*ry+oy, x+s*rx+ox] wt(o,i,ry,rx):
//                    the forward (s = -1) and the CONVERTED adjoint, the sheared
//                    gather d_input(x) += d_output(x + r.x) * kernel(r.x) with
//                    zero-padded d_output (s = +1, transposed k).
//                    32 x 16 output tile, input window of 8 channels and weights
//                    staged in shared memory, 2 px x 16 output channels per thread.
//   conv_dx_atomic   the unconverted scatter d_input(ro.y - ro.x) += d_output(ro.y) *
//                    kernel(ro.x) with red.global.add: the
//                    "general scatter with atomics" fallback.
//   conv_dk_partial  d_kernel = sum over pixels of dy x shifted x: persistent blocks,
//                    per-block partials in registers (thread = 4 output channels x one
//                    (ci, ry) x all rx; fp32 per 32-px tile row, fp64 across rows), then
//   conv_dk_finalize fixed-order fp64 sum of the block partials (deterministic).
#include "common.cuh"

namespace rs {
namespace {

constexpr int kCT = 256;
constexpr int kTX = 32, kTY = 16;  // output tile (thread = column, rows r and r + 8)
constexpr int kOB = 16;            // output channels per block (register block)
constexpr int kIB = 8;             // input channels per staged chunk

struct ConvDir {
    int O, I, s, oy, ox;
    long long so, si;  // wt(o, i, ry, rx) = k[o*so + i*si + ry*kw + rx]
};

__global__ void __launch_bounds__(kCT)
    conv_direct(const float *__restrict__ in, const float *__restrict__ k, float *__restrict__ out, int H, int W,
                int kh, int kw, ConvDir d, int tiles_x) {
    extern __shared__ __align__(16) float csm[];
    const int SH = kTY + kh - 1, SW = kTX + kw - 1, SP = SW + 1;
    float *sin = csm;                               // kIB x SH x SP
    float4 *swt = (float4 *)(sin + ((kIB * SH * SP + 3) & ~3));  // [i][ry][rx][kOB/4]
    const int n = blockIdx.y, og = blockIdx.z;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int x0 = tx * kTX, y0 = ty * kTY;
    const int col = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    const long long HW = (long long)H * W;
    // input window origin: positions y0 + yl + s*ry + oy over yl < kTY, ry < kh
    const int yb = d.s < 0 ? y0 + d.oy - (kh - 1) : y0 + d.oy;
    const int xb = d.s < 0 ? x0 + d.ox - (kw - 1) : x0 + d.ox;
    float acc[2][kOB];
#pragma unroll
    for (int o = 0; o < kOB; o++) acc[0][o] = acc[1][o] = 0.f;
    const float *inn = in + (long long)n * d.I * HW;
    for (int i0 = 0; i0 < d.I; i0 += kIB) {
        const int ni = min(kIB, d.I - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < ni * SH * SW; e += kCT) {
            const int ii = e / (SH * SW), rem = e - ii * (SH * SW);
            const int rr = rem / SW, cc = rem - rr * SW;
            const int gy = yb + rr, gx = xb + cc;
            float v = 0.f;
            if (gy >= 0 && gy < H && gx >= 0 && gx < W) v = __ldg(inn + (long long)(i0 + ii) * HW + (long long)gy * W + gx);
            sin[(ii * SH + rr) * SP + cc] = v;
        }
        const int nw = ni * kh * kw * (kOB / 4);
        for (int e = threadIdx.x; e < nw; e += kCT) {
            const int o4 = e % (kOB / 4), rest = e / (kOB / 4);
            const int r = rest % (kh * kw), ii = rest / (kh * kw);
            float w[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int o = og * kOB + 4 * o4 + t;
                w[t] = o < d.O ? __ldg(k + o * d.so + (i0 + ii) * d.si + r) : 0.f;
            }
            swt[rest * (kOB / 4) + o4] = make_float4(w[0], w[1], w[2], w[3]);
        }
        __syncthreads();
        for (int ii = 0; ii < ni; ii++) {
            for (int ry = 0; ry < kh; ry++) {
                const int wy = d.s < 0 ? kh - 1 - ry : ry;
                const float *s0 = sin + (ii * SH + r0 + wy) * SP + col;
                const float *s1 = s0 + 8 * SP;
                for (int rx = 0; rx < kw; rx++) {
                    const int wx = d.s < 0 ? kw - 1 - rx : rx;
                    const float v0 = s0[wx], v1 = s1[wx];
                    const float4 *wp = swt + ((ii * kh + ry) * kw + rx) * (kOB / 4);
#pragma unroll
                    for (int o4 = 0; o4 < kOB / 4; o4++) {
                        const float4 w = wp[o4];
                        acc[0][4 * o4 + 0] = fmaf(v0, w.x, acc[0][4 * o4 + 0]);
                        acc[0][4 * o4 + 1] = fmaf(v0, w.y, acc[0][4 * o4 + 1]);
                        acc[0][4 * o4 + 2] = fmaf(v0, w.z, acc[0][4 * o4 + 2]);
                        acc[0][4 * o4 + 3] = fmaf(v0, w.w, acc[0][4 * o4 + 3]);
                        acc[1][4 * o4 + 0] = fmaf(v1, w.x, acc[1][4 * o4 + 0]);
                        acc[1][4 * o4 + 1] = fmaf(v1, w.y, acc[1][4 * o4 + 1]);
                        acc[1][4 * o4 + 2] = fmaf(v1, w.z, acc[1][4 * o4 + 2]);
                        acc[1][4 * o4 + 3] = fmaf(v1, w.w, acc[1][4 * o4 + 3]);
                    }
                }
            }
        }
    }
    const int x = x0 + col;
    if (x >= W) return;
    float *outn = out + (long long)n * d.O * HW;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int y = y0 + r0 + 8 * h;
        if (y >= H) continue;
#pragma unroll
        for (int o = 0; o < kOB; o++) {
            const int oc = og * kOB + o;
            if (oc < d.O) outn[(long long)oc * HW + (long long)y * W + x] = acc[h][o];
        }
    }
}

// thread per (n, co, y, x): every tap of the gather becomes a red
__global__ void __launch_bounds__(kCT)
    conv_dx_atomic(const float *__restrict__ dy, const float *__restrict__ k, float *__restrict__ dx, int N, int Ci,
                   int Co, int H, int W, int kh, int kw) {
    const long long HW = (long long)H * W;
    const long long idx = (long long)blockIdx.x * kCT + threadIdx.x;
    if (idx >= (long long)N * Co * HW) return;
    const long long rem = idx % HW;
    const long long nc = idx / HW;
    const int co = (int)(nc % Co), n = (int)(nc / Co);
    const int y = (int)(rem / W), x = (int)(rem % W);
    const int ph = kh / 2, pw = kw / 2;
    const float g = __ldg(dy + idx);
    float *dxn = dx + (long long)n * Ci * HW;
    for (int ci = 0; ci < Ci; ci++) {
        const float *kp = k + ((long long)co * Ci + ci) * kh * kw;
        for (int ry = 0; ry < kh; ry++) {
            const int u = y - ry + ph;
            if (u < 0 || u >= H) continue;
            for (int rx = 0; rx < kw; rx++) {
                const int v = x - rx + pw;
                if (v < 0 || v >= W) continue;
                red_add(dxn + (long long)ci * HW + (long long)u * W + v, g * __ldg(kp + ry * kw + rx));
            }
        }
    }
}

constexpr int kKMax = 7;  // kw bound of the d_kernel register block

// Persistent blocks over (sample, 32 x 16 tile); task = (4 output channels, ci, ry):
// 4 x kw sums in registers across all the block's tiles, one partial per block.
__global__ void __launch_bounds__(kCT)
    conv_dk_partial(const float *__restrict__ x, const float *__restrict__ dy, double *__restrict__ part, int N, int Ci,
                    int Co, int H, int W, int kh, int kw, int tiles_x, int tiles) {
    extern __shared__ __align__(16) float csm[];
    const int SH = kTY + kh - 1, SW = kTX + kw - 1, SP = SW + 1;
    const int CO4 = (Co + 3) / 4;
    float4 *sg = (float4 *)csm;                  // [p][CO4] dy tile, 4 channels per float4
    float *sx = (float *)(sg + kTY * kTX * CO4);  // [ci][SH][SP] x window
    const int ph = kh / 2, pw = kw / 2;
    const long long HW = (long long)H * W;
    const int ntask = CO4 * Ci * kh;
    const int task = blockIdx.z * kCT + threadIdx.x;
    const bool act = task < ntask;
    const int cog = act ? task % CO4 : 0, rest = act ? task / CO4 : 0;
    const int ry = rest % kh, ci = rest / kh;
    // fp32 sums over one tile row (32 px), folded into fp64 sums per row: the rounding
    // of a 10^6-term sum stays far below the rms-scaled tolerance (Q14)
    double accd[4][kKMax];
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
        for (int r = 0; r < kKMax; r++) accd[t][r] = 0.0;
    const int per_sample = tiles;
    for (int tt = blockIdx.x; tt < N * per_sample; tt += gridDim.x) {
        const int n = tt / per_sample, tl = tt - n * per_sample;
        const int x0 = (tl % tiles_x) * kTX, y0 = (tl / tiles_x) * kTY;
        __syncthreads();
        // dy tile, transposed to [p][co]
        for (int e = threadIdx.x; e < CO4 * 4 * kTY * kTX; e += kCT) {
            const int co = e / (kTY * kTX), p = e - co * (kTY * kTX);
            const int yy = y0 + p / kTX, xx = x0 + p % kTX;
            float v = 0.f;
            if (co < Co && yy < H && xx < W) v = __ldg(dy + ((long long)n * Co + co) * HW + (long long)yy * W + xx);
            ((float *)sg)[p * CO4 * 4 + co] = v;
        }
        // x window: rows y0 + ph - (kh-1) .., columns x0 + pw - (kw-1) ..
        const int yb = y0 + ph - (kh - 1), xb = x0 + pw - (kw - 1);
        for (int e = threadIdx.x; e < Ci * SH * SW; e += kCT) {
            const int c = e / (SH * SW), r2 = e - c * (SH * SW);
            const int rr = r2 / SW, cc = r2 - rr * SW;
            const int gy = yb + rr, gx = xb + cc;
            float v = 0.f;
            if (gy >= 0 && gy < H && gx >= 0 && gx < W) v = __ldg(x + ((long long)n * Ci + c) * HW + (long long)gy * W + gx);
            sx[(c * SH + rr) * SP + cc] = v;
        }
        __syncthreads();
        if (act) {
            // pixel (yl, xl) reads x at window (yl + kh-1-ry, xl + kw-1-rx)
            const float *xr = sx + (ci * SH + (kh - 1 - ry)) * SP + (kw - 1);
            for (int yl = 0; yl < kTY; yl++) {
                float acc[4][kKMax];
#pragma unroll
                for (int t = 0; t < 4; t++)
#pragma unroll
                    for (int r = 0; r < kKMax; r++) acc[t][r] = 0.f;
                for (int xl = 0; xl < kTX; xl++) {
                    const float4 g = sg[(yl * kTX + xl) * CO4 + cog];
                    const float *xp = xr + yl * SP + xl;
#pragma unroll
                    for (int rx = 0; rx < kKMax; rx++) {
                        if (rx < kw) {
                            const float v = xp[-rx];
                            acc[0][rx] = fmaf(g.x, v, acc[0][rx]);
                            acc[1][rx] = fmaf(g.y, v, acc[1][rx]);
                            acc[2][rx] = fmaf(g.z, v, acc[2][rx]);
                            acc[3][rx] = fmaf(g.w, v, acc[3][rx]);
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < 4; t++)
#pragma unroll
                    for (int r = 0; r < kKMax; r++) accd[t][r] += (double)acc[t][r];
            }
        }
    }
    if (!act) return;
    const long long E = (long long)Co * Ci * kh * kw;
    double *pb = part + (long long)blockIdx.x * E;
#pragma unroll
    for (int t = 0; t < 4; t++) {
        const int co = 4 * cog + t;
        if (co >= Co) continue;
#pragma unroll
        for (int rx = 0; rx < kKMax; rx++)
            if (rx < kw) pb[(((long long)co * Ci + ci) * kh + ry) * kw + rx] = accd[t][rx];
    }
}

__global__ void conv_dk_finalize(const double *__restrict__ part, float *__restrict__ dk, int nb, long long E) {
    const long long e = (long long)blockIdx.x * kCT + threadIdx.x;
    if (e >= E) return;
    double s = 0.0;
    for (int b = 0; b < nb; b++) s += part[(long long)b * E + e];
    dk[e] = (float)s;
}

size_t direct_smem(int kh, int kw) {
    const int SH = kTY + kh - 1, SP = kTX + kw;
    return sizeof(float) * (((kIB * SH * SP + 3) & ~3) + (size_t)kIB * kh * kw * kOB);
}

size_t dk_smem(int Ci, int Co, int kh, int kw) {
    const int SH = kTY + kh - 1, SP = kTX + kw;
    return sizeof(float) * ((size_t)kTY * kTX * ((Co + 3) / 4) * 4 + (size_t)Ci * SH * SP);
}

int dk_blocks(int N, int H, int W) {
    const int tiles = ((W + kTX - 1) / kTX) * ((H + kTY - 1) / kTY);
    const long long total = (long long)N * tiles;
    return (int)(total < 296 ? total : 296);  // 2 per SM: partials stay small
}

cudaError_t launch_direct(const float *in, const float *k, float *out, int N, int H, int W, int kh, int kw,
                          const ConvDir &d, cudaStream_t s) {
    const int tiles_x = (W + kTX - 1) / kTX, tiles_y = (H + kTY - 1) / kTY;
    const size_t sm = direct_smem(kh, kw);
    if (sm > 48 * 1024) cudaFuncSetAttribute(conv_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    conv_direct<<<dim3(tiles_x * tiles_y, N, (d.O + kOB - 1) / kOB), kCT, sm, s>>>(in, k, out, H, W, kh, kw, d, tiles_x);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool conv_shape_ok(int Ci, int Co, int kh, int kw) {
    return kh >= 1 && kw >= 1 && kh <= kKMax && kw <= kKMax && dk_smem(Ci, Co, kh, kw) <= 200 * 1024;
}

size_t conv_ws_bytes(int N, int Ci, int Co, int H, int W, int kh, int kw) {
    return sizeof(double) * (size_t)dk_blocks(N, H, W) * Co * Ci * kh * kw;
}

cudaError_t conv_fwd_launch(const ConvArgs &a, cudaStream_t s) {
    ConvDir d;
    d.O = a.Co; d.I = a.Ci; d.s = -1; d.oy = a.kh / 2; d.ox = a.kw / 2;
    d.so = (long long)a.Ci * a.kh * a.kw; d.si = (long long)a.kh * a.kw;
    return launch_direct(a.x, a.k, a.y, a.N, a.H, a.W, a.kh, a.kw, d, s);
}

cudaError_t conv_bwd_launch(const ConvArgs &a, int algo, void *ws, size_t ws_bytes, cudaStream_t s) {
    const long long HW = (long long)a.H * a.W;
    if (a.dx) {
        if (algo == 3 /*SCATTER_ATOMIC*/) {
            cudaError_t e = cudaMemsetAsync(a.dx, 0, sizeof(float) * (size_t)a.N * a.Ci * HW, s);
            if (e != cudaSuccess) return e;
            const long long total = (long long)a.N * a.Co * HW;
            conv_dx_atomic<<<(unsigned)((total + kCT - 1) / kCT), kCT, 0, s>>>(a.dy, a.k, a.dx, a.N, a.Ci, a.Co,
                                                                               a.H, a.W, a.kh, a.kw);
            note_launch();
        } else {
            ConvDir d;  // sheared gather: out = dx (O = Ci), in = dy (I = Co), k transposed
            d.O = a.Ci; d.I = a.Co; d.s = 1; d.oy = -(a.kh / 2); d.ox = -(a.kw / 2);
            d.so = (long long)a.kh * a.kw; d.si = (long long)a.Ci * a.kh * a.kw;
            cudaError_t e = launch_direct(a.dy, a.k, a.dx, a.N, a.H, a.W, a.kh, a.kw, d, s);
            if (e != cudaSuccess) return e;
        }
    }
    if (a.dk) {
        if (ws_bytes < conv_ws_bytes(a.N, a.Ci, a.Co, a.H, a.W, a.kh, a.kw)) return cudaErrorInvalidValue;
        const int tiles_x = (a.W + kTX - 1) / kTX, tiles = tiles_x * ((a.H + kTY - 1) / kTY);
        const int nb = dk_blocks(a.N, a.H, a.W);
        const int ntask = ((a.Co + 3) / 4) * a.Ci * a.kh;
        const size_t sm = dk_smem(a.Ci, a.Co, a.kh, a.kw);
        if (sm > 48 * 1024) cudaFuncSetAttribute(conv_dk_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        double *part = (double *)ws;
        conv_dk_partial<<<dim3(nb, 1, (ntask + kCT - 1) / kCT), kCT, sm, s>>>(a.x, a.dy, part, a.N, a.Ci, a.Co, a.H,
                                                                              a.W, a.kh, a.kw, tiles_x, tiles);
        note_launch();
        const long long E = (long long)a.Co * a.Ci * a.kh * a.kw;
        conv_dk_finalize<<<(unsigned)((E + kCT - 1) / kCT), kCT, 0, s>>>(part, a.dk, nb, E);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace rs
