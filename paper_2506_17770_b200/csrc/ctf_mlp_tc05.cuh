// ctf_mlp_tc05.cuh — CTA-level collaboration for the latent-MLP format on the 5th-generation
// tensor cores (included by ctf_filter.cu in the latent-MLP translation unit).
//
// The paper's collaboration is per wave: a wave's lanes decode its n unique texels, at most one
// each.  For an expensive decoder the paper points at collaboration beyond one wave
// through shared memory (a "hybrid between wave communication and using shared
// memory"): here the four warps of a CTA pool the unique texels of their waves — every wave
// still evaluates exactly its own unique set (same records, evaluation counts and producers of
// the texels; only the hardware that runs the evaluations is shared) — and decode them as the
// rows of one tensor-core batch:
//   * round: each warp runs the lean front (a1-a4) of its next pair of waves (pair_front: the
//     exact unique set, ranks, jobs); the CTA concatenates the jobs (<= 4 x 64 rows);
//   * per 128 rows: row r's thread computes the 12 MLP inputs of its texel (R-10) and writes
//     them, split hi + lo in fp16 (3xFP16, R-29), to a shared-memory A tile (canonical
//     K-major core-matrix layout, no swizzle); one thread issues tcgen05.mma (M = 128, N = 32 /
//     32 / 16, K = 16 / 32 / 32; D in TMEM, fp32) for the three layers — hi*hi + hi*lo + lo*hi
//     per product, layer 1's bias folded in as an input column of 1.0 — and each thread moves
//     its row back with tcgen05.ld, applies bias / ReLU / clamp, and re-splits it into the next
//     layer's A tile;
//   * the decoded values (fp32 RGBA, row-indexed) go to a shared table; each warp gathers its
//     two waves' corners from it and blends (a6), exactly as the one-warp path does.
// Waves the lean front does not finish (n > 32, wide windows, partial or non-interior waves)
// are marked for the general kernel, as in the one-warp lean kernel.
#pragma once

namespace tc05 {

constexpr int kWarpsT = 8;            // warps per CTA: 256 threads, one row each of two 128-row tiles
constexpr int kTile = 128;            // rows per tensor-core tile (M)
constexpr int kIter = kWarpsT * 32;   // rows per decode iteration (two tiles, one MMA round trip)
constexpr int kMaxRows = kWarpsT * 64;   // jobs per round: <= 64 per warp (a pair of waves)

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tcgen05 shared-memory matrix descriptor, no swizzle: start >> 4, LBO (byte stride between
// core matrices adjacent along K) >> 4 at bit 16, SBO (byte stride between 8-row groups) >> 4
// at bit 32, version 1 at bit 46 (measured: scripts/probes/tc05_probe.cu).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor, kind::f16: D fp32 (bit 4), A / B fp16 K-major, N >> 3 at 17, M >> 4 at 24
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, bool acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)acc));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n\t}" ::"r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane (warp w reads lanes 32w..32w+31)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
// 16 fp32 values -> 16 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float4 (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(taddr), "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z),
                   "f"(v[1].w), "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z),
                   "f"(v[3].w)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __uint_as_float(r[j]);
}

// K-major core-matrix layout of an R x K fp16 matrix: 8 x 8 blocks of 128 B (row i of a block
// at +16 i), the K/8 blocks of an 8-row group contiguous (LBO = 128), groups (SBO = K/8 * 128)
__device__ __forceinline__ uint32_t cm_off(int r, int k8, int K) {
    return (uint32_t)(r >> 3) * (uint32_t)(K / 8) * 128u + (uint32_t)k8 * 128u + (uint32_t)(r & 7) * 16u;
}

struct alignas(1024) CtaSmem {
    uint32_t ah[kIter * 16], al[kIter * 16];   // A tiles hi / lo: 256 rows x 32 fp16 (layer 1: 16)
    uint32_t w1h[32 * 8], w1l[32 * 8];          // B1 [32][16]: W1 | b1 column | 0
    uint32_t w2h[32 * 16], w2l[32 * 16];        // B2 [32][32]
    uint32_t w3h[16 * 16], w3l[16 * 16];        // B3 [16][32]: rows 4..15 zero
    float b2[32], b3[4];
    float4 xch[kMaxRows];                       // job row -> decoded RGBA
    uint8_t bits[kWarpsT][96];                  // per warp: job -> window offset (pair_front; 64..95 scratch)
    int info[kWarpsT][8];                       // per warp: jobs, nA, A.minx, A.miny, B.minx, B.miny
    unsigned long long mbar;
    uint32_t tmem;
};

// rows of fp16 halves: 8 halves (16 B) of row r, K-chunk k8 of a K-wide tile
__device__ __forceinline__ void st_chunk(uint32_t *base, int r, int k8, int K, uint4 v) {
    *reinterpret_cast<uint4 *>(reinterpret_cast<unsigned char *>(base) + cm_off(r, k8, K)) = v;
}

// weights -> B operands (hi / lo fp16, K-major core-matrix layout), once per CTA
__device__ __forceinline__ void fill_weights(const MlpWeights &mw, CtaSmem &s) {
    const float *o = mw.v;   // kernel layout: W1[j][k], b1, W2T[k][j], b2, W3T[j][c], b3
    auto put = [](uint32_t *h, uint32_t *l, int n, int k, int K, float x0, float x1) {
        uint32_t hh, ll;
        split2(x0, x1, hh, ll);
        const uint32_t off = cm_off(n, k >> 3, K) + (uint32_t)(k & 7) * 2u;
        *reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(h) + off) = hh;
        *reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(l) + off) = ll;
    };
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) {   // B1[n][k], k = 2i'..: W1, then b1 at k = 12
        const int n = i >> 3, k = 2 * (i & 7);
        auto val = [&](int kk) { return kk < 12 ? o[n * 12 + kk] : kk == 12 ? o[384 + n] : 0.f; };
        put(s.w1h, s.w1l, n, k, 16, val(k), val(k + 1));
    }
    for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) {  // B2[n][k] = W2T[k][n]
        const int n = i >> 4, k = 2 * (i & 15);
        put(s.w2h, s.w2l, n, k, 32, o[416 + k * 32 + n], o[416 + (k + 1) * 32 + n]);
    }
    for (int i = threadIdx.x; i < 16 * 16; i += blockDim.x) {  // B3[n][k] = W3T[k][n], n < 4
        const int n = i >> 4, k = 2 * (i & 15);
        put(s.w3h, s.w3l, n, k, 32, n < 4 ? o[1472 + k * 4 + n] : 0.f, n < 4 ? o[1472 + (k + 1) * 4 + n] : 0.f);
    }
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
        s.b2[i] = o[1440 + i];
        if (i < 4) s.b3[i] = o[1600 + i];
    }
}

// one layer's MMAs on the current A tile: D[128 x N] (+)= A * B^T with 3xFP16 (hi*hi, hi*lo,
// lo*hi).  Descriptors are built once per CTA; the K step of 16 (two core matrices, 256 B)
// advances the start address field (bits 0-13, in 16-B units) by 16.
struct Descs {
    uint64_t ah16, al16, ah32, al32, w1h, w1l, w2h, w2l, w3h, w3l;
};
__device__ __forceinline__ Descs make_descs(const CtaSmem &s) {
    Descs d;
    d.ah16 = umma_desc(smem_addr(s.ah), 128u, 256u);
    d.al16 = umma_desc(smem_addr(s.al), 128u, 256u);
    d.ah32 = umma_desc(smem_addr(s.ah), 128u, 512u);
    d.al32 = umma_desc(smem_addr(s.al), 128u, 512u);
    d.w1h = umma_desc(smem_addr(s.w1h), 128u, 256u);
    d.w1l = umma_desc(smem_addr(s.w1l), 128u, 256u);
    d.w2h = umma_desc(smem_addr(s.w2h), 128u, 512u);
    d.w2l = umma_desc(smem_addr(s.w2l), 128u, 512u);
    d.w3h = umma_desc(smem_addr(s.w3h), 128u, 512u);
    d.w3l = umma_desc(smem_addr(s.w3l), 128u, 512u);
    return d;
}
// tile t of an iteration: A rows 128t.. (16 row groups further: 16 * K/8 * 128 B), accumulator
// columns 32t..
template <int K, int N>
__device__ __forceinline__ void layer_mma(uint32_t tmem, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, bool acc,
                                          int ntiles) {
    constexpr uint32_t idesc = umma_idesc(kTile, N);
    constexpr uint64_t tile_step = 16u * (K / 8) * 128u / 16u;   // in 16-B units
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        if (t >= ntiles) break;
        const uint32_t d = tmem + 32u * (uint32_t)t;
        const uint64_t to = (uint64_t)t * tile_step;
#pragma unroll
        for (int kk = 0; kk < K / 16; ++kk) {
            const uint64_t ko = (uint64_t)kk * 16u;
            umma_f16(d, ah + to + ko, bh + ko, idesc, acc || kk > 0);
            umma_f16(d, ah + to + ko, bl + ko, idesc, true);
            umma_f16(d, al + to + ko, bh + ko, idesc, true);
        }
    }
}

}  // namespace tc05

// The CTA-level kernel (release build, latent MLP, COLLAB List / Box / Mask, no forced fallback).
template <bool GRAD, bool BOX>
__global__ void __launch_bounds__(tc05::kWarpsT * 32, CTF_TC05_MINB)
    ctf_mlp_tc05_kernel(const __grid_constant__ KArgs a, const MlpWeights mw) {
    using namespace tc05;
    extern __shared__ __align__(1024) unsigned char dyn_raw[];
    CtaSmem &s = *reinterpret_cast<CtaSmem *>(dyn_raw + ((1024u - (smem_addr(dyn_raw) & 1023u)) & 1023u));
    const unsigned lane = lane_id(), warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);
    const unsigned tid = threadIdx.x, lt_mask = lanemask_lt();
    fill_weights(mw, s);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s.tmem)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s.mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = s.tmem, mbar = smem_addr(&s.mbar);
    // this thread's row: tile warp / 4 (accumulator columns 32 (warp / 4)..), TMEM lane 32 (warp % 4) + lane
    const uint32_t trow = tmem + (((warp & 3u) * 32u) << 16) + 32u * (warp >> 2);
    uint32_t phase = 0u;
    const Descs dsc = make_descs(s);
    // one thread issues a layer's MMAs, commits them to the mbarrier and waits for it; the
    // CTA barrier then releases the other threads (blocked warps do not issue)
    int ntiles = 1;   // tiles of the current iteration (1 or 2)
    auto run_layer = [&](int layer) {
        if (tid == 0) {
            tc_after_sync();
            if (layer == 1) layer_mma<16, 32>(tmem, dsc.ah16, dsc.al16, dsc.w1h, dsc.w1l, false, ntiles);
            else if (layer == 2) layer_mma<32, 32>(tmem, dsc.ah32, dsc.al32, dsc.w2h, dsc.w2l, true, ntiles);   // bias pre-stored
            else layer_mma<32, 16>(tmem, dsc.ah32, dsc.al32, dsc.w3h, dsc.w3l, false, ntiles);
            umma_commit(mbar);
            mbar_wait(mbar, phase);
        }
        phase ^= 1u;
        __syncthreads();
        tc_after_sync();
    };

    const int lx = (int)(lane & 7), ly = (int)(lane >> 3);
    struct XchRef { float4 *xch; } xr{s.xch};
    // per-warp run state
    unsigned k = 0;                      // item counter of this warp
    unsigned c = 0;                      // current item
    int fr = 0, wy = 0, wx0 = 0, wx1 = 0, wx = 0, py = 0;
    unsigned pix = 0, w0 = 0;
    uint32_t frame = 0, myrec = 0;
    bool have = false;
    float2 uv_a = make_float2(0.f, 0.f), uv_b = uv_a;
    uint2 gr_a = make_uint2(0u, 0u), gr_b = gr_a;
    const unsigned stride_items = gridDim.x * kWarpsT;
    // claim the next interior run (non-interior runs: every wave to the general kernel)
    auto next_item = [&]() {
        have = false;
        for (;;) {
            c = blockIdx.x * kWarpsT + warp + k * stride_items;
            if (c >= a.nchunks) return;
            ++k;
            fr = (int)(c / (unsigned)a.cpf);
            const int rr = (int)(c - (unsigned)fr * (unsigned)a.cpf);
            wy = rr / a.cpr;
            wx0 = (rr - wy * a.cpr) * a.chunk;
            wx1 = min(wx0 + a.chunk, a.nwx);
            py = wy * 4 + ly;
            frame = a.frame_index + (uint32_t)fr;
            w0 = (unsigned)fr * (unsigned)a.wpf + (unsigned)(wy * a.nwx + wx0);
            pix = (unsigned)fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)(wx0 * 8 + lx);
            const bool interior = wy * 4 + 4 <= a.Hf && wx1 * 8 <= a.Wf;
            if (interior) {
                wx = wx0;
                myrec = 0u;
                uv_a = uv_b = make_float2(__int_as_float(0x7fc00000), 0.f);
                gr_a = gr_b = make_uint2(0u, 0u);
                ld_stream_f2_if(uv_a, a.uv + pix, true);
                ld_stream_u2_if(gr_a, a.grad + pix, GRAD);
                ld_stream_f2_if(uv_b, a.uv + (pix + 8u), wx0 + 1 < wx1);
                ld_stream_u2_if(gr_b, a.grad + (pix + 8u), (wx0 + 1 < wx1) & GRAD);
                have = true;
                return;
            }
            // non-interior run: records say "general path", appended to its work list
            const bool inrun = lane < (unsigned)(wx1 - wx0);
            if (inrun) a.rec[w0 + lane] = kSlowMark;
            const unsigned msl = __ballot_sync(FULL, inrun);
            if (a.lists) {
                const unsigned b1 = __shfl_sync(FULL, atom_add_if(a.lcnt + 1, (unsigned)__popc(msl), lane == 0), 0);
                st_u32_if(a.lists + a.nrec + b1 + __popc(msl & lt_mask), w0 + lane, inrun);
            }
        }
    };
    next_item();
    for (;;) {
        // ---- fronts: this warp's next pair (A, B) of its run; jobs -> bits, counts -> info
        PairFront fa, fb;
        fa.n = fb.n = 0;
        fa.rec = fb.rec = 0u;
        const bool hasB = have && wx + 1 < wx1;
        if (have) {
            fa = pair_front<GRAD, FMT_MLP, XchRef, BOX>(a, xr, uv_a, gr_a, 0, s.bits[warp], lane, lt_mask, push_codes(lane));
            __syncwarp();
            if (hasB) fb = pair_front<GRAD, FMT_MLP, XchRef, BOX>(a, xr, uv_b, gr_b, fa.n, s.bits[warp], lane, lt_mask, push_codes(lane));
            // next pair's inputs
            uv_a = uv_b = make_float2(__int_as_float(0x7fc00000), 0.f);
            gr_a = gr_b = make_uint2(0u, 0u);
            ld_stream_f2_if(uv_a, a.uv + (pix + 16u), wx + 2 < wx1);
            ld_stream_u2_if(gr_a, a.grad + (pix + 16u), (wx + 2 < wx1) & GRAD);
            ld_stream_f2_if(uv_b, a.uv + (pix + 24u), wx + 3 < wx1);
            ld_stream_u2_if(gr_b, a.grad + (pix + 24u), (wx + 3 < wx1) & GRAD);
        }
        if (lane == 0) {
            s.info[warp][0] = fa.n + fb.n;
            s.info[warp][1] = fa.n;
            s.info[warp][2] = fa.minx;
            s.info[warp][3] = fa.miny;
            s.info[warp][4] = fb.minx;
            s.info[warp][5] = fb.miny;
        }
        const int any = __syncthreads_or(have ? 1 : 0);
        if (!any) break;
        int base[kWarpsT + 1];
        base[0] = 0;
#pragma unroll
        for (int w = 0; w < kWarpsT; ++w) base[w + 1] = base[w] + s.info[w][0];
        const int T = base[kWarpsT];
        // ---- decode the round's jobs, 128 rows per tensor-core tile
        for (int t0 = 0; t0 < T; t0 += kIter) {
            ntiles = T - t0 > kTile ? 2 : 1;
            const int row = t0 + (int)tid;
            if (row < T) {   // this thread's row: locate its wave's job, compute the 12 inputs (R-10)
                int w = 0;
                int bw = 0;
#pragma unroll
                for (int q = 1; q < kWarpsT; ++q) {
                    const bool ge = row >= base[q];
                    w += ge ? 1 : 0;
                    bw = ge ? base[q] : bw;
                }
                const int j = row - bw;
                const int nA = s.info[w][1];
                const uint32_t e = s.bits[w][j];
                const int qx = (j < nA ? s.info[w][2] : s.info[w][4]) + (int)(e & 7u);
                const int qy = (j < nA ? s.info[w][3] : s.info[w][5]) + (int)(e >> 3);
                float in[12];
                mlp_features(a.tex, qx, qy, in);
                uint32_t h[8], l[8];
#pragma unroll
                for (int q = 0; q < 6; ++q) split2(in[2 * q], in[2 * q + 1], h[q], l[q]);
                h[6] = 0x3C00u;   // (1.0, 0): layer 1's bias column
                l[6] = 0u;
                h[7] = l[7] = 0u;
                st_chunk(s.ah, (int)tid, 0, 16, make_uint4(h[0], h[1], h[2], h[3]));
                st_chunk(s.ah, (int)tid, 1, 16, make_uint4(h[4], h[5], h[6], h[7]));
                st_chunk(s.al, (int)tid, 0, 16, make_uint4(l[0], l[1], l[2], l[3]));
                st_chunk(s.al, (int)tid, 1, 16, make_uint4(l[4], l[5], l[6], l[7]));
            }
            fence_async_smem();
            __syncthreads();
            run_layer(1);   // layer 1: 12 (+ bias column) -> 32
            // epilogue 1 / 2: ReLU, re-split into the next layer's A tile (K = 32); after layer 1
            // the row's accumulator is re-initialised with b2 (tcgen05.st) so layer 2 adds onto it
            const bool my_tile = (int)(warp >> 2) < ntiles;   // warp-uniform: this warp's tile was decoded
#pragma unroll 1
            for (int layer = 1; layer <= 2; ++layer) {
#pragma unroll
                for (int hlf = 0; hlf < 2; ++hlf) {
                    if (!my_tile) break;
                    float v[16];
                    tmem_ld16(trow + 16u * (uint32_t)hlf, v);
                    if (layer == 1) {
                        const float4 *b = reinterpret_cast<const float4 *>(s.b2) + 4 * hlf;
                        const float4 bv[4] = {b[0], b[1], b[2], b[3]};
                        tmem_st16(trow + 16u * (uint32_t)hlf, bv);
                    }
                    uint32_t h[8], l[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) split2(fmaxf(v[2 * q], 0.f), fmaxf(v[2 * q + 1], 0.f), h[q], l[q]);
                    st_chunk(s.ah, (int)tid, 2 * hlf, 32, make_uint4(h[0], h[1], h[2], h[3]));
                    st_chunk(s.ah, (int)tid, 2 * hlf + 1, 32, make_uint4(h[4], h[5], h[6], h[7]));
                    st_chunk(s.al, (int)tid, 2 * hlf, 32, make_uint4(l[0], l[1], l[2], l[3]));
                    st_chunk(s.al, (int)tid, 2 * hlf + 1, 32, make_uint4(l[4], l[5], l[6], l[7]));
                }
                if (layer == 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                fence_async_smem();
                tc_before_sync();
                __syncthreads();
                run_layer(layer + 1);   // layer 2: 32 -> 32 (onto b2); layer 3: 32 -> 4 (N = 16)
            }
            // epilogue 3: + b3, clamp [0, 1] -> the row's texel value
            if (my_tile) {
                float v[4];
                tmem_ld4(trow, v);
                if (row < T)
                    s.xch[row] = make_float4(fminf(fmaxf(v[0] + s.b3[0], 0.f), 1.f), fminf(fmaxf(v[1] + s.b3[1], 0.f), 1.f),
                                             fminf(fmaxf(v[2] + s.b3[2], 0.f), 1.f), fminf(fmaxf(v[3] + s.b3[3], 0.f), 1.f));
            }
            tc_before_sync();
        }
        __syncthreads();
        // ---- backs: gather + blend this warp's two waves from the round's table (a6)
        if (have) {
            int bw = 0;
#pragma unroll
            for (int q = 1; q < kWarpsT; ++q) bw = warp == (unsigned)q ? base[q] : bw;
            const uint32_t shift = 16u * (uint32_t)bw;
            fa.a0 += shift;
            fa.a2 += shift;
            fb.a0 += shift;
            fb.a2 += shift;
            pair_back(a, s, fa, pix);
            if (hasB) pair_back(a, s, fb, pix + 8u);
            if (lane == (unsigned)(wx - wx0)) myrec = fa.rec;
            if (lane == (unsigned)(wx + 1 - wx0)) myrec = hasB ? fb.rec : myrec;
            wx += 2;
            pix += 16u;
            if (wx >= wx1) {   // run done: records, work-list appends, next run
                const bool inrun = lane < (unsigned)(wx1 - wx0);
                if (inrun) a.rec[w0 + lane] = myrec;
                const unsigned msl = __ballot_sync(FULL, inrun && myrec == kSlowMark);
                if (a.lists && msl) {
                    const unsigned b1 = __shfl_sync(FULL, atom_add_if(a.lcnt + 1, (unsigned)__popc(msl), lane == 0), 0);
                    st_u32_if(a.lists + a.nrec + b1 + __popc(msl & lt_mask), w0 + lane, (msl >> lane) & 1u);
                }
                next_item();
            }
        }
        __syncwarp();
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}
