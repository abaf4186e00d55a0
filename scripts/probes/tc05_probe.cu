// tcgen05 probe: D[128 x N] (fp32, TMEM) = A[128 x K] * B[N x K]^T (fp16, K-major, smem, no swizzle)
// Tries the descriptor conventions (which of LBO / SBO strides K vs M/N) and prints the max error
// of each variant against a host reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>

constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version (sm100)
    return d;                  // base offset 0, swizzle none (bits 61-63 = 0)
}

// core-matrix layout: element (r, k) of an R x K (K-major) matrix at
//   (r / 8) * rstride + (k / 8) * kstride + (r % 8) * 16 + (k % 8) * 2 bytes
__device__ __forceinline__ uint32_t cm_off(int r, int k, uint32_t rstride, uint32_t kstride) {
    return (uint32_t)(r >> 3) * rstride + (uint32_t)(k >> 3) * kstride + (uint32_t)(r & 7) * 16u + (uint32_t)(k & 7) * 2u;
}

__global__ void probe(const __half *A, const __half *B, float *D, int variant) {
    __shared__ __align__(1024) unsigned char sA[M * K * 2];
    __shared__ __align__(1024) unsigned char sB[N * K * 2];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // layout: layout 0 = k-groups contiguous inside a row group (kstride 128, rstride K/8*128)
    //         layout 1 = row groups contiguous inside a k group (rstride 128, kstride R/8*128)
    const int layout = variant >> 1, swap = variant & 1;
    const uint32_t a_r = layout == 0 ? (K / 8) * 128u : 128u, a_k = layout == 0 ? 128u : (M / 8) * 128u;
    const uint32_t b_r = layout == 0 ? (K / 8) * 128u : 128u, b_k = layout == 0 ? 128u : (N / 8) * 128u;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__half *>(sA + cm_off(r, k, a_r, a_k)) = A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__half *>(sB + cm_off(r, k, b_r, b_k)) = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int kk = 0; kk < K / 16; ++kk) {
            // K step of 16 = two core matrices along K
            const uint32_t ao = kk * 2 * a_k, bo = kk * 2 * b_k;
            const uint64_t da = swap ? make_desc(smem_u32(sA) + ao, a_r, a_k) : make_desc(smem_u32(sA) + ao, a_k, a_r);
            const uint64_t db = swap ? make_desc(smem_u32(sB) + bo, b_r, b_k) : make_desc(smem_u32(sB) + bo, b_k, b_r);
            const uint32_t acc = kk > 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMA
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(&mbar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 32; ++j) D[row * N + j] = __uint_as_float(v[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
    __half hA[M * K], hB[N * K];
    float fA[M * K], fB[N * K], ref[M * N];
    for (int i = 0; i < M * K; ++i) { fA[i] = (float)((i * 37 % 29) - 14) / 16.0f; hA[i] = __float2half(fA[i]); }
    for (int i = 0; i < N * K; ++i) { fB[i] = (float)((i * 53 % 31) - 15) / 8.0f; hB[i] = __float2half(fB[i]); }
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < N; ++c) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)fA[r * K + k] * fB[c * K + k];
            ref[r * N + c] = (float)s;
        }
    __half *dA, *dB;
    float *dD;
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, sizeof(ref));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 4; ++variant) {
        cudaMemset(dD, 0, sizeof(ref));
        probe<<<1, 128>>>(dA, dB, dD, variant);
        cudaError_t e = cudaDeviceSynchronize();
        float D[M * N];
        cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(D[i] - ref[i]));
        printf("variant %d (layout %d, %s): %s max err %.3g  D[0..3] %g %g %g %g ref %g %g %g %g\n", variant, variant >> 1,
               (variant & 1) ? "LBO=M/N stride" : "LBO=K stride", cudaGetErrorString(e), err, D[0], D[1], D[2], D[3],
               ref[0], ref[1], ref[2], ref[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
