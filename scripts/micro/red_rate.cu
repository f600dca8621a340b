// Microbenchmark: global float reduction throughput, scalar red.global.add.f32 vs
// vector red.global.add.v2/.v4.f32, spread addresses (each lane its own 16-B slot,
// a 256 MB target so lines miss L2 like the warp adjoint).  Prints G lane-ops/s and
// G floats/s.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(float *dst, size_t nslots, int iters) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t slot = (t * 2654435761u) % nslots;
    for (int it = 0; it < iters; it++) {
        float *p = dst + slot * 4;
        if (V == 1) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(1.f) : "memory");
        if (V == 2) asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(1.f) : "memory");
        if (V == 4) asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
        slot = (slot + 1) % nslots;  // consecutive lanes -> consecutive slots (coalesced-ish)
    }
}
// same, but lanes of a warp hit consecutive floats (scalar) like the warp layer's taps
__global__ void kc(float *dst, size_t n, int iters) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t i = (t * 37) % n;
    for (int it = 0; it < iters; it++) {
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + i), "f"(1.f) : "memory");
        i = (i + 4096) % n;
    }
}
int main() {
    const size_t bytes = 256ull << 20, nslots = bytes / 16;
    float *d; cudaMalloc(&d, bytes); cudaMemset(d, 0, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, iters = 64;
    const double ops = (double)blocks * threads * iters;
    auto run = [&](const char *name, auto kern, int floats) {
        kern<<<blocks, threads>>>(d, nslots, iters);
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) kern<<<blocks, threads>>>(d, nslots, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-22s %8.1f G lane-ops/s  %8.1f G floats/s\n", name, 5 * ops / (ms * 1e-3) / 1e9,
               5 * ops * floats / (ms * 1e-3) / 1e9);
    };
    run("red.f32 (16B slots)", k<1>, 1);
    run("red.v2.f32", k<2>, 2);
    run("red.v4.f32", k<4>, 4);
    kc<<<blocks, threads>>>(d, bytes / 4, iters);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) kc<<<blocks, threads>>>(d, bytes / 4, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-22s %8.1f G lane-ops/s\n", "red.f32 warp-contig", 5 * ops / (ms * 1e-3) / 1e9);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
