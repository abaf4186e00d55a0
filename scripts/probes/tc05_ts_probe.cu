// tcgen05 TS mode probe: A (128 x 32 fp16) written to TMEM by its row threads (tcgen05.st, two
// fp16 per 32-bit column, k ascending), B (32 x 32) from smem (K-major core matrices);
// D = A * B^T checked against the host.  Also times nmma TS MMAs.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
constexpr int M = 128, N = 32, K = 32;
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__global__ void k(const __half *A, const __half *B, float *D, long long *cyc, int nmma) {
    __shared__ __align__(1024) unsigned char sB[N * K * 2];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, c = i % K;
        *reinterpret_cast<__half *>(sB + (r >> 3) * (K / 8) * 128 + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2) = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tb)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tb;
    // row tid of A -> TMEM lane tid, columns 32..47 (16 words = 32 halves)
    uint32_t w[16];
    for (int c = 0; c < 16; ++c) {
        __half2 h = __halves2half2(A[tid * K + 2 * c], A[tid * K + 2 * c + 1]);
        w[c] = *reinterpret_cast<uint32_t *>(&h);
    }
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 32u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                   "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        long long t0 = clock64();
        for (int rep = 0; rep < nmma / 2; ++rep)
            for (int kk = 0; kk < 2; ++kk) {
                const uint64_t db = desc(sa(sB) + kk * 256, 128, 512);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(tm), "r"(tm + 32u + 8u * kk), "l"(db), "r"(idesc), "r"(kk > 0 ? 1 : 0));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&mbar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(sa(&mbar)), "r"(0) : "memory");
        cyc[0] = clock64() - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) D[tid * N + j] = __uint_as_float(v[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(64));
}
int main() {
    static __half hA[M * K], hB[N * K];
    static float fA[M * K], fB[N * K], ref[M * N], D[M * N];
    for (int i = 0; i < M * K; ++i) { fA[i] = (float)((i * 37 % 29) - 14) / 16.0f; hA[i] = __float2half(fA[i]); }
    for (int i = 0; i < N * K; ++i) { fB[i] = (float)((i * 53 % 31) - 15) / 8.0f; hB[i] = __float2half(fB[i]); }
    for (int r = 0; r < M; ++r) for (int c = 0; c < N; ++c) { double s = 0; for (int q = 0; q < K; ++q) s += (double)fA[r * K + q] * fB[c * K + q]; ref[r * N + c] = (float)s; }
    __half *dA, *dB; float *dD; long long *dc;
    cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, sizeof(D)); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    for (int nmma : {2, 12, 30, 60}) {
        k<<<1, 128>>>(dA, dB, dD, dc, nmma);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
        double err = 0; for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(D[i] - ref[i]));
        printf("TS nmma=%2d: %s err %.3g, %lld cycles (%.1f per MMA)\n", nmma, cudaGetErrorString(e), err, c, (double)c / nmma);
    }
    return 0;
}
