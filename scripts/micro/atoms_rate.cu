// shared-memory atomic add throughput on sm_100a: int32 / int64 ATOMS vs LDS+STS RMW,
// conflict-free (lane-consecutive) and 2-way / random patterns.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int *out, int iters, int stride) {
    __shared__ long long s64[4096];
    int *s32 = (int *)s64;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s64[i] = 0;
    __syncthreads();
    unsigned idx = (threadIdx.x * stride) & 4095u;
    int acc = 0;
    for (int it = 0; it < iters; it++) {
        const unsigned a = (idx + it * 97u) & 4095u;
        if (MODE == 0) atomicAdd(s32 + a, (int)(a ^ it));
        else if (MODE == 1) atomicAdd((unsigned long long *)(s64 + (a & 4095u)), 1ull);
        else if (MODE == 2) { s32[a] += 1; }
        else acc += s32[a];
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s32[threadIdx.x] + acc;
}
int main() {
    int *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    const int iters = 4096;
    const char *names[] = {"atoms.add.s32", "atoms.add.u64", "lds+sts (rmw)", "lds"};
    for (int stride : {1, 2, 33}) {
        for (int m = 0; m < 4; m++) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            auto launch = [&]() {
                if (m == 0) k<0><<<148 * 8, 256>>>(o, iters, stride);
                if (m == 1) k<1><<<148 * 8, 256>>>(o, iters, stride);
                if (m == 2) k<2><<<148 * 8, 256>>>(o, iters, stride);
                if (m == 3) k<3><<<148 * 8, 256>>>(o, iters, stride);
            };
            launch(); cudaDeviceSynchronize();
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double ops = 148.0 * 8 * 256 * iters;
            printf("stride %2d %-16s %8.3f ms  %7.1f G lane-ops/s  %5.2f lane-ops/clk/SM\n", stride, names[m], ms,
                   ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
