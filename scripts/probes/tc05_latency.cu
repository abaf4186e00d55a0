// tcgen05 round-trip latency: one thread issues n MMAs (M=128, N=32, K=16, SS), commits to an
// mbarrier and waits; clock64 from before the first issue to the wait's completion.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__global__ void k(long long *out, int nmma, int N) {
    __shared__ __align__(1024) unsigned char sA[128 * 32 * 2], sB[64 * 32 * 2];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tb;
    for (int i = threadIdx.x; i < (int)sizeof(sA) / 4; i += blockDim.x) ((uint32_t *)sA)[i] = 0x3C003C00u;
    for (int i = threadIdx.x; i < (int)sizeof(sB) / 4; i += blockDim.x) ((uint32_t *)sB)[i] = 0x3C003C00u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tb)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint64_t da = desc(sa(sA), 128, 512), db = desc(sa(sB), 128, 512);
        for (int rep = 0; rep < 4; ++rep) {
            long long t0 = clock64();
            for (int i = 0; i < nmma; ++i) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tb), "l"(da + (uint64_t)((i & 1) * 16)), "l"(db), "r"(idesc), "r"(i > 0 ? 1 : 0));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&mbar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(sa(&mbar)), "r"(rep & 1) : "memory");
            long long t1 = clock64();
            if (rep == 3) out[0] = t1 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(64));
}
int main() {
    long long *d; cudaMalloc(&d, 8);
    for (int N : {16, 32, 64}) for (int n : {1, 3, 6, 12, 30, 60}) {
        k<<<1, 128>>>(d, n, N);
        long long h = 0; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%d nmma=%2d: %lld cycles (%.1f per MMA) %s\n", N, n, h, (double)h / n, cudaGetErrorString(e));
    }
    return 0;
}
