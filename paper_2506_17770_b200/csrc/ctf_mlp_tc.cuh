// ctf_mlp_tc.cuh — the tensor-core latent-MLP texel decoder shared by the bilinear and the
// bicubic kernels (included inside namespace ctf after ctf_device.cuh).
#pragma once

// ------------------------------------- tensor-core latent-MLP decode
// The wave's texels (one per lane: row = lane) go through the three layers as
// mma.sync m16n8k16 tiles (M = 32 texels in 2 tiles, fp32 accumulate).  fp16 operands
// would round weights and activations to 11 bits, so every operand is split into
// hi = fp16(x) and lo = fp16(x - hi) and each product is formed as
// hi*hi + hi*lo + lo*hi (3 MMAs, the classic 3xFP16 scheme): ~22-bit operands, fp32
// accumulation, measured |error| <= 3e-7 against the fp64 oracle (R-29) — far inside
// the 1e-5 parity bar, with no fp16 rounding decision anywhere.  A layer's C fragment
// (rows g, g+8; columns 2q, 2q+1) is exactly the next layer's A fragment, so the
// activations never leave registers; only the 12 inputs and 4 outputs pass through
// shared memory.
struct TcWeights {          // per CTA, filled once from the kernel-parameter weights
    uint32_t w1h[32][12], w1l[32][12];   // W1[n][k] as half2 words (k padded 12 -> 16, row stride 24 halfs)
    uint32_t w2h[32][20], w2l[32][20];   // W2[n][k] (row stride 40 halfs: conflict-free fragment loads)
    uint32_t w3h[8][20], w3l[8][20];     // W3[n][k], rows 4..7 zero
    float b1[32], b2[32], b3[8];
};
struct TcScratch {          // per warp
    uint32_t ah[32][12], al[32][12];     // layer-1 inputs as half2 words (row = texel = lane)
    float4 out[32];
};

// split a pair (x0, x1) into hi / lo half2 words: hi = fp16(x) (one packed cvt), the
// residual x - hi is exact in fp32 (one fma.f32.f16 each), lo = fp16(residual)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t &h, uint32_t &l) {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
    const float r0 = fma_f32_f16((unsigned short)(h & 0xffffu), (unsigned short)0xBC00u, x0);   // x0 - hi0
    const float r1 = fma_f32_f16((unsigned short)(h >> 16), (unsigned short)0xBC00u, x1);
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(r1), "f"(r0));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// four 8x8 b16 matrices from shared memory, lane i addressing row i % 8 of matrix i / 8;
// register j of lane t = matrix j, row t / 4, columns 2 (t % 4), +1: the mma fragment layout
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"((unsigned)__cvta_generic_to_shared(p))
                 : "memory");
}
// d += A * B with A = Ah + Al, B = Bh + Bl, dropping Al * Bl (3xFP16)
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t bh0,
                                     uint32_t bh1, uint32_t bl0, uint32_t bl1) {
    mma16816(d, ah, bh0, bh1);
    mma16816(d, ah, bl0, bl1);
    mma16816(d, al, bh0, bh1);
}

// kernel-layout weights (W1[j][k], b1, W2T[k][j], b2, W3T[j][c], b3) -> TcWeights, by all threads
__device__ __forceinline__ void fill_tc_weights(const MlpWeights &mw, TcWeights &tw) {
    const float *o = mw.v;
    for (int i = threadIdx.x; i < 32 * 12; i += blockDim.x) {       // W1: n = i / 12, word = i % 12
        const int n = i / 12, w = i % 12, k = 2 * w;
        const float x0 = k < 12 ? o[n * 12 + k] : 0.f, x1 = k + 1 < 12 ? o[n * 12 + k + 1] : 0.f;
        split2(x0, x1, tw.w1h[n][w], tw.w1l[n][w]);
    }
    for (int i = threadIdx.x; i < 32 * 20; i += blockDim.x) {       // W2[n][k] = W2T[k][n]
        const int n = i / 20, w = i % 20, k = 2 * w;
        const float x0 = k < 32 ? o[416 + k * 32 + n] : 0.f, x1 = k + 1 < 32 ? o[416 + (k + 1) * 32 + n] : 0.f;
        split2(x0, x1, tw.w2h[n][w], tw.w2l[n][w]);
    }
    for (int i = threadIdx.x; i < 8 * 20; i += blockDim.x) {        // W3[n][k] = W3T[k][n]
        const int n = i / 20, w = i % 20, k = 2 * w;
        const float x0 = (n < 4 && k < 32) ? o[1472 + k * 4 + n] : 0.f;
        const float x1 = (n < 4 && k + 1 < 32) ? o[1472 + (k + 1) * 4 + n] : 0.f;
        split2(x0, x1, tw.w3h[n][w], tw.w3l[n][w]);
    }
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
        tw.b1[i] = o[384 + i];
        tw.b2[i] = o[1440 + i];
        if (i < 8) tw.b3[i] = i < 4 ? o[1600 + i] : 0.f;
    }
}

// Decode texel (qx, qy) of every lane with `valid` set; returns this lane's texel.
__device__ __forceinline__ float4 mlp_decode_tc(const TexArgs &t, const TcWeights &tw, TcScratch &sm, bool valid,
                                                int qx, int qy, unsigned lane) {
    {
        float in[12];
        if (valid) {
            mlp_features(t, qx, qy, in);
        } else {
#pragma unroll
            for (int k = 0; k < 12; ++k) in[k] = 0.f;
        }
#pragma unroll
        for (int w = 0; w < 6; ++w) split2(in[2 * w], in[2 * w + 1], sm.ah[lane][w], sm.al[lane][w]);
        sm.ah[lane][6] = sm.ah[lane][7] = 0u;
        sm.al[lane][6] = sm.al[lane][7] = 0u;
    }
    __syncwarp();
    const int g = (int)(lane >> 2), q = (int)(lane & 3);
    const int nmt = __any_sync(FULL, valid && lane >= 16) ? 2 : 1;   // rows 16..31 unused -> one M tile
    float out[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        if (mt >= nmt) break;
        // fragments by ldmatrix: lane i addresses row (i & 7) of matrix mi = i >> 3
        const int mi = (int)(lane >> 3), mr = (int)(lane & 7);
        uint32_t ah[4], al[4];   // rows 16mt + (mi & 1) * 8 + mr, words (mi >> 1) * 4 ..
        ldsm_x4(ah, &sm.ah[16 * mt + (mi & 1) * 8 + mr][(mi >> 1) * 4]);
        ldsm_x4(al, &sm.al[16 * mt + (mi & 1) * 8 + mr][(mi >> 1) * 4]);
        // layer 1: 12 (16) -> 32, ReLU; C fragments become layer-2 A fragments (k-tiles of 16)
        uint32_t a2h[2][4], a2l[2][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int c = 8 * nt + 2 * q;
            float d[4] = {tw.b1[c], tw.b1[c + 1], tw.b1[c], tw.b1[c + 1]};
            uint32_t b[4];   // {hi b0, hi b1, lo b0, lo b1} of W1 rows 8nt..8nt+7
            ldsm_x4(b, &((mi & 2) ? tw.w1l : tw.w1h)[8 * nt + mr][(mi & 1) * 4]);
            mma3(d, ah, al, b[0], b[1], b[2], b[3]);
            const int kt = nt >> 1, hi = nt & 1;
            split2(fmaxf(d[0], 0.f), fmaxf(d[1], 0.f), a2h[kt][2 * hi], a2l[kt][2 * hi]);
            split2(fmaxf(d[2], 0.f), fmaxf(d[3], 0.f), a2h[kt][2 * hi + 1], a2l[kt][2 * hi + 1]);
        }
        // layer 2: 32 -> 32, ReLU
        uint32_t a3h[2][4], a3l[2][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int c = 8 * nt + 2 * q;
            float d[4] = {tw.b2[c], tw.b2[c + 1], tw.b2[c], tw.b2[c + 1]};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                uint32_t b[4];
                ldsm_x4(b, &((mi & 2) ? tw.w2l : tw.w2h)[8 * nt + mr][8 * kt + (mi & 1) * 4]);
                mma3(d, a2h[kt], a2l[kt], b[0], b[1], b[2], b[3]);
            }
            const int kt = nt >> 1, hi = nt & 1;
            split2(fmaxf(d[0], 0.f), fmaxf(d[1], 0.f), a3h[kt][2 * hi], a3l[kt][2 * hi]);
            split2(fmaxf(d[2], 0.f), fmaxf(d[3], 0.f), a3h[kt][2 * hi + 1], a3l[kt][2 * hi + 1]);
        }
        // layer 3: 32 -> 4 (8 columns, 4..7 zero), clamp [0, 1]
        {
            const int c = 2 * q;
            float d[4] = {tw.b3[c], tw.b3[c + 1], tw.b3[c], tw.b3[c + 1]};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                uint32_t b[4];
                ldsm_x4(b, &((mi & 2) ? tw.w3l : tw.w3h)[mr][8 * kt + (mi & 1) * 4]);
                mma3(d, a3h[kt], a3l[kt], b[0], b[1], b[2], b[3]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) out[mt][i] = fminf(fmaxf(d[i], 0.f), 1.f);
        }
    }
    // rows r0 (cols 2q, 2q+1) and r0 + 8 of each tile -> the texel's lane; q < 2 hold RGBA
    float *o = reinterpret_cast<float *>(sm.out);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        if (mt >= nmt || q >= 2) continue;
        const int r0 = 16 * mt + g;
        *reinterpret_cast<float2 *>(o + 4 * r0 + 2 * q) = make_float2(out[mt][0], out[mt][1]);
        *reinterpret_cast<float2 *>(o + 4 * (r0 + 8) + 2 * q) = make_float2(out[mt][2], out[mt][3]);
    }
    __syncwarp();
    const float4 v = sm.out[lane];
    __syncwarp();
    return v;
}

