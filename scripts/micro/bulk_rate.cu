// Microbenchmark: HBM->smem streaming with TMA bulk copies of S bytes vs cp.async 16 B.
// Each block streams its slice of a large buffer through a 2-stage smem ring; consumers
// read one float per 16 B so the data is used.  Prints GB/s per (mode, S).
#include <cstdio>
#include <cuda_runtime.h>
#define DEV __device__ __forceinline__
DEV unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
DEV void mb_init(unsigned long long *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
DEV void mb_tx(unsigned long long *b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
DEV void bulk(void *d, const void *s, unsigned n, unsigned long long *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
DEV bool mb_try(unsigned long long *b, unsigned ph) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
    return ok;
}
DEV void cpa16(void *d, const void *s) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d)), "l"(s) : "memory"); }

constexpr int STAGE = 16384;  // bytes per stage
template <int MODE>
__global__ void __launch_bounds__(256) k(const char *src, size_t per_block, int S, float *out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ unsigned long long bar[2];
    const char *base = src + blockIdx.x * per_block;
    const int nst = (int)(per_block / STAGE);
    if (threadIdx.x == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    float acc = 0.f;
    auto issue = [&](int st) {
        char *d = sm + (st & 1) * STAGE;
        const char *s = base + (size_t)st * STAGE;
        if (MODE == 0) {
            if (threadIdx.x == 0) mb_tx(&bar[st & 1], STAGE);
            for (int o = threadIdx.x * S; o < STAGE; o += 256 * S) bulk(d + o, s + o, S, &bar[st & 1]);
        } else {
            for (int o = threadIdx.x * 16; o < STAGE; o += 256 * 16) cpa16(d + o, s + o);
            asm volatile("cp.async.commit_group;");
        }
    };
    issue(0);
    for (int st = 0; st < nst; st++) {
        if (st + 1 < nst) issue(st + 1);
        if (MODE == 0) { while (!mb_try(&bar[st & 1], (st >> 1) & 1)) {} }
        else { if (st + 1 < nst) asm volatile("cp.async.wait_group 1;"); else asm volatile("cp.async.wait_group 0;"); __syncthreads(); }
        const float *f = (const float *)(sm + (st & 1) * STAGE);
        for (int i = threadIdx.x; i < STAGE / 4; i += 256) acc += f[i];
        __syncthreads();
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    const size_t total = 2ull << 30;
    char *src; float *out;
    cudaMalloc(&src, total); cudaMalloc(&out, 4);
    cudaMemset(src, 0, total);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int bps : {2, 3, 4}) {
        const int blocks = 148 * bps;
        const size_t per = (total / blocks) / STAGE * STAGE;
        for (int mode = 0; mode < 2; mode++) {
            for (int S : {64, 128, 256, 512, 2048}) {
                if (mode == 1 && S != 64) continue;
                auto kern = mode == 0 ? k<0> : k<1>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * STAGE);
                kern<<<blocks, 256, 2 * STAGE>>>(src, per, S, out);
                cudaEventRecord(e0);
                for (int r = 0; r < 3; r++) kern<<<blocks, 256, 2 * STAGE>>>(src, per, S, out);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                printf("blocks/SM %d %s S=%4d: %.0f GB/s\n", bps, mode ? "cp.async16" : "bulk", mode ? 16 : S,
                       3.0 * per * blocks / (ms * 1e-3) / 1e9);
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
