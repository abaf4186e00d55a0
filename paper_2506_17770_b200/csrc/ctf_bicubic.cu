// ctf_bicubic.cu — collaborative filtering with the bicubic filters of §5.4
// ("Bicubic Filtering"): cubic B-spline and Catmull-Rom, 4x4 footprints,
// <= 1 or <= 2 texel evaluations per lane on the exact path (Fig. 13).
//
// Same wave model as the bilinear kernel (one 8x4 wave per warp), with:
//   a2  footprint: taps x0-1..x0+2 / y0-1..y0+2 clamped (R-24), weights R-25, clamp
//       duplicates merged per axis -> an nc x nr grid of distinct cells per lane;
//   a3  collect: the wave's distinct texels in ascending id on a 32 x 32 shared-memory bitmap
//       of the wave's AABB (one word per row; each lane ORs its nc-bit column run into its nr
//       rows with shared atomics): n = sum of the row popcounts, a texel's rank = exclusive
//       scan of the row counts + popc within its row (a lane's cells in a row have
//       consecutive ranks), each texel's first setter publishes rank -> id.  AABBs wider than
//       32 x 32 (minified waves) "peel" instead: one redux.sync.min per distinct texel;
//       the record's n saturates at E*a + 1 (R-28);
//   a4  exact iff n <= E*a (List), AABB area <= E*a (Box), AABB <= MxM and n <= E*a (Mask);
//   a5  rank r is produced by lane h(r mod a, A) as its (r div a)-th evaluation;
//   a6  16 shared-memory reads of the produced fp32 values by rank + the 16-cell FFMA2 chain;
//   a7  fallbacks STF / C / C+ with |w|-proportional one-tap samples (R-26);
//   STF mode: the positivized two-lobe estimator (R-27).
// Independent of oracle/.  P:n = PAPER.md line; R-n = DESIGN.md reading.
#include <climits>
#include <cstdint>

#include "ctf_device.cuh"
#include "ctf_internal.h"

#ifndef CTF_TU_FMT
#define CTF_TU_FMT 1
#endif

namespace ctf {
namespace {

#include "ctf_mlp_tc.cuh"

constexpr int kBWarps = 8;
constexpr int kBChunk = 16;  // waves per work item (a run in one wave-row)
enum { FILT_BSPLINE = 1, FILT_CATMULL_ROM = 2 };
enum { BVAR_LIST = 0, BVAR_BOX = 1, BVAR_MASK16 = 2, BVAR_MASK11 = 3 };

struct BArgs {
    TexArgs tex;
    const float2 *uv;
    const uint2 *grad;
    float4 *out;
    uint32_t *rec;
    unsigned fpx;
    int Wf, Hf, nwx, nwy, wpf, cpr, cpf;
    unsigned nchunks, ipw;
    float Wflt, Hflt;
    int filter, E, fallback, variant;
    uint32_t flags, frame_index, seed_lo, seed_hi;
    int row0;                       // RNG counter y = row0 + py (strip sharding)
};

struct BSmem {
    uint32_t tbl[128];        // exact: rank -> (y << 16) | x (ranks >= 124 clamped: unused); C+: sorted planned ids
    uint32_t sorted[32];      // fallback gather: sorted (id << 5 | lane) of produced texels
    uint32_t bm[32];          // collect: AABB bitmap, one word per row
    float4 xch[64];           // exact: rank -> produced value (fp32)
    uint8_t lane_of_rank[32]; // h(r, A)
};

// ------------------------------------------------------------------ weights (R-25)
// fp32, one rounding per operation in the written order (no contraction): they decide
// integers (STF / C+ picks), so the oracle computes the identical values.
__device__ __forceinline__ void cubic_weights(int filter, float s, float (&w)[4]) {
    const float r = __fsub_rn(1.0f, s);
    const float s2 = __fmul_rn(s, s), s3 = __fmul_rn(s2, s), r2 = __fmul_rn(r, r);
    if (filter == FILT_BSPLINE) {
        w[0] = __fdiv_rn(__fmul_rn(r2, r), 6.0f);
        w[1] = __fdiv_rn(__fadd_rn(__fsub_rn(__fmul_rn(3.0f, s3), __fmul_rn(6.0f, s2)), 4.0f), 6.0f);
        w[2] = __fdiv_rn(__fadd_rn(__fadd_rn(__fsub_rn(__fmul_rn(3.0f, s2), __fmul_rn(3.0f, s3)), __fmul_rn(3.0f, s)),
                                   1.0f),
                         6.0f);
        w[3] = __fdiv_rn(s3, 6.0f);
    } else {
        w[0] = __fmul_rn(-0.5f, __fmul_rn(s, r2));
        w[1] = __fmul_rn(__fadd_rn(__fsub_rn(__fmul_rn(3.0f, s3), __fmul_rn(5.0f, s2)), 2.0f), 0.5f);
        w[2] = __fmul_rn(__fadd_rn(__fsub_rn(__fmul_rn(4.0f, s2), __fmul_rn(3.0f, s3)), s), 0.5f);
        w[3] = __fmul_rn(-0.5f, __fmul_rn(s2, r));
    }
}

// One lane's 4x4 footprint (R-24): distinct columns xa..xa+nc-1, rows ya..ya+nr-1,
// merged weights per distinct column / row (taps in ascending order).
struct Foot16 {
    int xa, nc, ya, nr;
    float wx[4], wy[4];   // tap weights
    float mx[4], my[4];   // merged (0 beyond nc / nr)
    int cx[4], ry[4];     // tap -> distinct column / row index
};

__device__ __forceinline__ void merge_axis(const float (&w)[4], const int (&idx)[4], float (&m)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (idx[i] == c) acc = __fadd_rn(acc, w[i]);
        m[c] = acc;
    }
}

// fx = fma(clamp(u), W, -0.5) -> (x0, s); shared with the C+ spare-lane recomputation.
// interior (warp-uniform: every lane's 4 x 4 taps inside the texture): no clamp duplicates,
// merged weight c = 0 + w_c (the bits merge_axis adds)
__device__ __forceinline__ Foot16 footprint16(int filter, int x0, int y0, float s, float t, int W, int H,
                                              bool interior = false) {
    Foot16 f;
    cubic_weights(filter, s, f.wx);
    cubic_weights(filter, t, f.wy);
    f.xa = min(max(x0 - 1, 0), W - 1);
    f.ya = min(max(y0 - 1, 0), H - 1);
    const int xb = min(max(x0 + 2, 0), W - 1), yb = min(max(y0 + 2, 0), H - 1);
    f.nc = xb - f.xa + 1;
    f.nr = yb - f.ya + 1;
    if (interior) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f.cx[i] = i;
            f.ry[i] = i;
            f.mx[i] = __fadd_rn(0.0f, f.wx[i]);
            f.my[i] = __fadd_rn(0.0f, f.wy[i]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f.cx[i] = min(max(x0 - 1 + i, 0), W - 1) - f.xa;
            f.ry[i] = min(max(y0 - 1 + i, 0), H - 1) - f.ya;
        }
        merge_axis(f.wx, f.cx, f.mx);
        merge_axis(f.wy, f.ry, f.my);
    }
    return f;
}

__device__ __forceinline__ float sel4(const float (&v)[4], int i) {
    return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
}
__device__ __forceinline__ int sel4i(const int (&v)[4], int i) { return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3]; }

// the 16-cell blend: acc over cells (r outer, c inner) of fma((mx[c] * my[r]), v, acc) with the
// texel values v in fp32 ([0, 1]: Texel::to_f4, R-9 / R-10), two channels per FFMA2.  The
// exact path, the full filter and Eq. 1's "all known" case use this one chain, so exact waves
// equal the full filter bit for bit.
struct Acc {
    uint64_t rg, ba;
    __device__ __forceinline__ Acc() : rg(0ull), ba(0ull) {}
    __device__ __forceinline__ void add(float w, const float4 &v) {
        rg = ffma2(f2pack(v.x, v.y), f2pack(w, w), rg);
        ba = ffma2(f2pack(v.z, v.w), f2pack(w, w), ba);
    }
    __device__ __forceinline__ float4 get() const {
        const float2 a = f2unpack(rg), b = f2unpack(ba);
        return make_float4(a.x, a.y, b.x, b.y);
    }
};

// R-26: index of the tap drawn with probability |w_i| / S (fp32 inverse CDF)
__device__ __forceinline__ int cubic_pick(const float (&w)[4], float u, float &S) {
    S = 0.0f;
    int last = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        S = __fadd_rn(S, fabsf(w[i]));
        if (w[i] != 0.0f) last = i;
    }
    const float target = __fmul_rn(u, S);
    float cum = 0.0f;
    int pick = -1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cum = __fadd_rn(cum, fabsf(w[i]));
        if (pick < 0 && cum > target) pick = i;
    }
    return pick < 0 ? last : pick;
}

__device__ __forceinline__ int eq2_rank(int j, int np, int na) {  // Eq. 2, R-18
    if (np >= na - 1) return 0;
    return (2 * (na - 1) * (j - np) + (na - 1 - np)) / (2 * (na - 1 - np));
}

// MODE (4TAP / STF / COLLAB), the filter and Box sampling are compile-time (one instantiation
// each): the exact collaborative path compiles to straight-line code
template <int FMT, int MODE, int FILT, bool BOX>
#ifndef CTF_BIC_MINB
#define CTF_BIC_MINB 4  // BC1 bicubic kernel: resident CTAs per SM (64 registers; 3: 76 registers, -9 %)
#endif
#ifndef CTF_BIC_MLP_MINB
#define CTF_BIC_MLP_MINB 4  // latent-MLP bicubic kernel: resident CTAs per SM (64 registers, small spills: 2.15x over 1 CTA / 167 registers)
#endif
__global__ void __launch_bounds__(kBWarps * 32, FMT == FMT_BC1 ? CTF_BIC_MINB : CTF_BIC_MLP_MINB)
    ctf_bicubic_kernel(const BArgs a, const typename WeightsOf<FMT>::type mw) {
    __shared__ BSmem smem[kBWarps];
    const unsigned lane = lane_id(), warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);   // provably warp-uniform (no divergence guards)
    BSmem &s = smem[warp];
    // finite values in every exchange slot: the exact gather reads cells beyond a lane's
    // clamped footprint with weight 0 (no select)
    s.xch[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    s.xch[lane + 32] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    // latent MLP, collaborative: the texels a wave produces are decoded together on the tensor
    // cores (mlp_decode_tc, rows = lanes, R-29), the weights staged once per CTA
    constexpr bool TC = FMT == FMT_MLP && MODE == MODE_COLLAB;
    extern __shared__ __align__(16) unsigned char bic_dyn[];
    TcWeights *tw = nullptr;
    TcScratch *tsc = nullptr;
    if constexpr (TC) {
        tw = reinterpret_cast<TcWeights *>(bic_dyn);
        tsc = &reinterpret_cast<TcScratch *>(bic_dyn + sizeof(TcWeights))[warp];
        fill_tc_weights(mw, *tw);
        __syncthreads();
    }
    const int lx = (int)(lane & 7), ly = (int)(lane >> 3);
    const unsigned lt = lanemask_lt();
    const int W = a.tex.W, H = a.tex.H;

    for (unsigned j = 0; j < a.ipw; ++j) {
        const unsigned c = (blockIdx.x * kBWarps + warp) + j * gridDim.x * kBWarps;
        if (c >= a.nchunks) break;
        const int fr = (int)(c / (unsigned)a.cpf);
        const int rr = (int)(c - (unsigned)fr * (unsigned)a.cpf);
        const int wy = rr / a.cpr;
        const int wx0 = (rr - wy * a.cpr) * kBChunk;
        const int wx1 = min(wx0 + kBChunk, a.nwx);
        const int py = wy * 4 + ly;
        const uint32_t frame = a.frame_index + (uint32_t)fr;
        for (int wx = wx0; wx < wx1; ++wx) {
            const int px = wx * 8 + lx;
            const bool inframe = py < a.Hf && px < a.Wf;
            const unsigned pix = (unsigned)fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)px;
            const unsigned widx = (unsigned)fr * (unsigned)a.wpf + (unsigned)(wy * a.nwx + wx);
            float2 uv = make_float2(__int_as_float(0x7fc00000), 0.0f);
            uint2 gr = make_uint2(0u, 0u);
            if (inframe) {
                uv = ld_stream_f2(a.uv + pix);
                if (a.grad) gr = ld_stream_u2(a.grad + pix);
            }
            __syncwarp();
            // ---- a1: classify
            const bool active = inframe && !isnan(uv.x);
            const unsigned A = __ballot_sync(FULL, active);
            const int na = __popc(A);
            if (na == 0) {
                if (inframe) st_stream_f4(a.out + pix, make_float4(0.f, 0.f, 0.f, 0.f));
                if (lane == 0) a.rec[widx] = ((MODE == MODE_COLLAB ? 0u : 0xFFu) << 8) | (1u << 26);
                continue;
            }
            bool mag_lane = true;
            if (a.grad && active) {
                const float rx = fma_f32_f16((unsigned short)(gr.x & 0xffffu), (unsigned short)(gr.x & 0xffffu),
                                             fma_f32_f16((unsigned short)(gr.x >> 16), (unsigned short)(gr.x >> 16), 0.0f));
                const float ry = fma_f32_f16((unsigned short)(gr.y & 0xffffu), (unsigned short)(gr.y & 0xffffu),
                                             fma_f32_f16((unsigned short)(gr.y >> 16), (unsigned short)(gr.y >> 16), 0.0f));
                mag_lane = rx <= 1.0f && ry <= 1.0f;
            }
            const bool wave_mag = a.grad != nullptr && __all_sync(FULL, mag_lane);
            const int ar = __popc(A & lt);
            if (active) s.lane_of_rank[ar] = (uint8_t)lane;
            // ---- a2: footprint (R-24, R-25)
            const float fx = fmaf(__saturatef(uv.x), a.Wflt, -0.5f), fy = fmaf(__saturatef(uv.y), a.Hflt, -0.5f);
            const float flx = floorf(fx), fly = floorf(fy);
            const int x0 = (int)flx, y0 = (int)fly;
            const float fs = __fsub_rn(fx, flx), ft = __fsub_rn(fy, fly);
            const bool interior = __all_sync(FULL, !active || (x0 >= 1 && x0 + 2 <= W - 1 && y0 >= 1 && y0 + 2 <= H - 1));
            const Foot16 f = footprint16(FILT, x0, y0, fs, ft, W, H, interior);
            __syncwarp();

            float4 color = make_float4(0.f, 0.f, 0.f, 0.f);
            int evals = 0, n = 0xFF, path = 0;
            int run_fb = -1;
            if (MODE == MODE_4TAP) {
                // the full filter: every lane evaluates its 16 taps (cells; clamp duplicates
                // are evaluated once per tap in the count, once per cell here)
                Acc acc;
#pragma unroll 1
                for (int q = 0; q < 16; ++q) {
                    const int r = q >> 2, cc = q & 3;
                    const bool valid = active && r < f.nr && cc < f.nc;
                    Texel<FMT> v = Texel<FMT>::zero();
                    if (valid) v = produce(a.tex, mw, (uint32_t)(f.xa + cc), (uint32_t)(f.ya + r));
                    acc.add(__fmul_rn(sel4(f.mx, cc), sel4(f.my, r)), v.to_f4());
                }
                color = acc.get();
                evals = 16 * na;
                path = PATH_4TAP;
            } else if (MODE == MODE_STF) {
                // R-27 positivized STF: one draw per lobe, c = W+ p+ - W- p-
                const uint4 rnd = philox4x32_10(make_uint4((uint32_t)px, (uint32_t)(py + a.row0), frame, 0u), a.seed_lo, a.seed_hi);
                float Wp = 0.0f, Wn = 0.0f;
                int lastp = 0, lastn = 0;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const float w = __fmul_rn(f.wx[k & 3], f.wy[k >> 2]);
                    if (w > 0.0f) { Wp = __fadd_rn(Wp, w); lastp = k; }
                    else if (w < 0.0f) { Wn = __fadd_rn(Wn, -w); lastn = k; }
                }
                int pk[2];
#pragma unroll
                for (int lobe = 0; lobe < 2; ++lobe) {
                    const float Wl = lobe ? Wn : Wp;
                    const float target = __fmul_rn(unit24(lobe ? rnd.y : rnd.x), Wl);
                    float cum = 0.0f;
                    int pick = -1;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float w = __fmul_rn(f.wx[k & 3], f.wy[k >> 2]);
                        const bool in = lobe ? (w < 0.0f) : (w > 0.0f);
                        if (in) {
                            cum = __fadd_rn(cum, lobe ? -w : w);
                            if (pick < 0 && cum > target) pick = k;
                        }
                    }
                    pk[lobe] = pick < 0 ? (lobe ? lastn : lastp) : pick;
                }
                float cc4[4] = {0.f, 0.f, 0.f, 0.f};
                const bool two = Wn > 0.0f;
#pragma unroll 1
                for (int lobe = 0; lobe < 2; ++lobe) {
                    if (!__any_sync(FULL, active && (lobe == 0 || two))) break;
                    const bool need = active && (lobe == 0 || two);
                    const int k = pk[lobe];
                    Texel<FMT> v = Texel<FMT>::zero();
                    if (need)
                        v = produce(a.tex, mw, (uint32_t)(f.xa + sel4i(f.cx, k & 3)), (uint32_t)(f.ya + sel4i(f.ry, k >> 2)));
                    const float4 e = v.to_f4();
                    const float Wl = lobe ? -Wn : Wp;
                    cc4[0] = need ? fmaf(Wl, e.x, cc4[0]) : cc4[0];
                    cc4[1] = need ? fmaf(Wl, e.y, cc4[1]) : cc4[1];
                    cc4[2] = need ? fmaf(Wl, e.z, cc4[2]) : cc4[2];
                    cc4[3] = need ? fmaf(Wl, e.w, cc4[3]) : cc4[3];
                }
                color = make_float4(cc4[0], cc4[1], cc4[2], cc4[3]);
                evals = __reduce_add_sync(FULL, active ? (two ? 2 : 1) : 0);
                path = PATH_STF;
            } else {
                // ---- a3: collect (ascending id; ranks of the lane's row starts)
                const int E = a.E;
                const int limit = E * na + 1;
                const int minx = __reduce_min_sync(FULL, active ? f.xa : INT_MAX);
                const int miny = __reduce_min_sync(FULL, active ? f.ya : INT_MAX);
                const int maxx = __reduce_max_sync(FULL, active ? f.xa + f.nc - 1 : INT_MIN);
                const int maxy = __reduce_max_sync(FULL, active ? f.ya + f.nr - 1 : INT_MIN);
                const int bw = maxx - minx + 1, bh = maxy - miny + 1;
                int rr[4] = {0, 0, 0, 0};
                int count = 0;
                if (bw <= 32 && bh <= 32) {
                    // bitmap of the AABB: row r = word r; a lane's cells in a row are the nc
                    // consecutive bits from xa - minx, so its ranks in that row are consecutive
                    s.bm[lane] = 0u;
                    __syncwarp();
                    const int cx = (f.xa - minx) & 31, cy = (f.ya - miny) & 31;
                    const uint32_t pat = ((1u << f.nc) - 1u) << cx;
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (active && r < f.nr) atomicOr(&s.bm[(cy + r) & 31], pat);
                    __syncwarp();
                    const uint32_t cnt = __popc(s.bm[lane]);
                    const int nx = (int)__reduce_add_sync(FULL, cnt);
                    uint32_t base = cnt;   // inclusive scan of the row counts (shfl.up's in-range
                                           // predicate guards the add: two instructions per step)
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1)
                        asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 u;\n\t"
                                     "shfl.sync.up.b32 u|p, %0, %1, 0, 0xffffffff;\n\t@p add.u32 %0, %0, u;\n\t}"
                                     : "+r"(base) : "r"(d));
                    base -= cnt;
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t b = __shfl_sync(FULL, base, (cy + r) & 31);
                        const uint32_t word = s.bm[(cy + r) & 31];
                        rr[r] = (int)b + __popc(word & ((1u << cx) - 1u));
                        // every lane publishes rank -> (y << 16) | x for each of its cells: a texel's rank
                        // and value do not depend on the lane, so lanes sharing a texel store the same
                        // word (ranks < E*a + 1 matter; the packed coordinates order like ids, W, H <=
                        // 2^16; a row starting at rank >= 124 only occurs in fallback waves, skipped)
                        const uint32_t v0 = ((uint32_t)(f.ya + r) << 16) | (uint32_t)f.xa;
                        if (interior) {   // 4 x 4 cells: one predicate per row, 4 stores off one address
                            if (active && rr[r] < 124) {
                                uint32_t *t = s.tbl + rr[r];
                                t[0] = v0;
                                t[1] = v0 + 1u;
                                t[2] = v0 + 2u;
                                t[3] = v0 + 3u;
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                if (active && r < f.nr && c < f.nc && rr[r] < 124) s.tbl[rr[r] + c] = v0 + (uint32_t)c;
                        }
                    }
                    count = nx < limit ? nx : limit;
                } else {
                    // wider than the bitmap: peel, one redux.sync.min per distinct texel
                    int r = 0, cc = 0;
                    uint32_t cur = active ? ((uint32_t)f.ya << 16) | (uint32_t)f.xa : INVALID_ID;
                    while (count < limit) {
                        const uint32_t m = __reduce_min_sync(FULL, cur);
                        if (m == INVALID_ID) break;
                        if (lane == 0) s.tbl[count] = m;
                        if (cur == m) {
                            if (cc == 0) {
                                rr[0] = r == 0 ? count : rr[0];
                                rr[1] = r == 1 ? count : rr[1];
                                rr[2] = r == 2 ? count : rr[2];
                                rr[3] = r == 3 ? count : rr[3];
                            }
                            if (++cc == f.nc) { cc = 0; ++r; }
                            cur = (r < f.nr) ? ((uint32_t)(f.ya + r) << 16) | (uint32_t)(f.xa + cc) : INVALID_ID;
                        }
                        ++count;
                    }
                }
                n = count;  // exact when <= E*a, else saturated at E*a + 1 (R-28)
                // ---- a4: decide
                bool ok;
                if (BOX) ok = bw * bh <= E * na;
                else if (a.variant == BVAR_MASK16) ok = bw <= 16 && bh <= 16 && n <= E * na;
                else if (a.variant == BVAR_MASK11) ok = bw <= 11 && bh <= 11 && n <= E * na;
                else ok = n <= E * na;
                if (a.flags & FLAG_FORCE_FALLBACK) ok = false;
                __syncwarp();
                if (ok) {
                    // ---- a5: produce (<= E per lane): rank i on lane h(i mod a, A), slot i div a;
                    // the value goes to the shared table by rank (fp32, converted once)
                    constexpr bool box = BOX;
                    const int total = box ? bw * bh : n;
#pragma unroll 1
                    for (int slot = 0; slot < 2; ++slot) {
                        if (slot * na >= total) break;
                        const int i = ar + slot * na;
                        const bool valid = active && i < total;
                        uint32_t tx = (uint32_t)minx, ty = (uint32_t)miny;
                        if (valid) {
                            if (box) {
                                ty = (uint32_t)(miny + i / bw);
                                tx = (uint32_t)(minx + i % bw);
                            } else {
                                const uint32_t e = s.tbl[i];
                                ty = e >> 16;
                                tx = e & 0xFFFFu;
                            }
                        }
                        if constexpr (TC) {
                            const float4 v = mlp_decode_tc(a.tex, *tw, *tsc, valid, (int)tx, (int)ty, lane);
                            if (valid) s.xch[i] = v;
                        } else {
                            if (valid) s.xch[i] = produce(a.tex, mw, tx, ty).to_f4();
                        }
                    }
                    __syncwarp();
                    // ---- a6: gather by rank + the 16-cell chain (bit-identical to the full filter)
                    Acc acc;
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int rq = q >> 2, cq = q & 3;
                        int rank;
                        if (box) rank = (f.ya + rq - miny) * bw + (f.xa + cq - minx);
                        else rank = rr[rq] + cq;
                        // a cell beyond the lane's clamped footprint (cq >= nc or rq >= nr) has merged
                        // weight 0 and reads a finite slot: fma(v, 0, acc) = acc, as the full filter's
                        // zero texel
                        const float4 v = s.xch[rank & 63];
                        acc.add(__fmul_rn(f.mx[cq], f.my[rq]), v);
                    }
                    color = acc.get();
                    evals = total;
                    path = PATH_EXACT;
                } else {
                    run_fb = a.fallback;
                    path = PATH_FB_STF + a.fallback;
                }
            }

            if (run_fb >= 0) {
                // ---- a7: fallbacks; one-tap plan (R-26)
                const uint4 rnd = philox4x32_10(make_uint4((uint32_t)px, (uint32_t)(py + a.row0), frame, 0u), a.seed_lo, a.seed_hi);
                float Sx, Sy;
                const int pi = cubic_pick(f.wx, unit24(rnd.x), Sx);
                const int pj = cubic_pick(f.wy, unit24(rnd.y), Sy);
                const int qx = f.xa + sel4i(f.cx, pi), qy = f.ya + sel4i(f.ry, pj);
                if (run_fb == FB_STF) {
                    Texel<FMT> v = Texel<FMT>::zero();
                    if (active) v = produce(a.tex, mw, (uint32_t)qx, (uint32_t)qy);
                    const float4 e = v.to_f4();
                    const bool neg = (sel4(f.wx, pi) < 0.0f) != (sel4(f.wy, pj) < 0.0f);
                    const float g = __fmul_rn(Sx, Sy) * (neg ? -1.0f : 1.0f);
                    color = make_float4(e.x * g, e.y * g, e.z * g, e.w * g);
                    evals = na;
                } else {
                    uint32_t prod = active ? (uint32_t)qy * (uint32_t)W + (uint32_t)qx : INVALID_ID;
                    if (run_fb == FB_CPLUS) {
                        // C+ (P:485-518): planned ids deduplicated ascending on lanes h(i, A) ...
                        const uint32_t sk = warp_sort32(prod);
                        const uint32_t skp = __shfl_up_sync(FULL, sk, 1);
                        const bool firstp = sk != INVALID_ID && (lane == 0 || sk != skp);
                        const unsigned F = __ballot_sync(FULL, firstp);
                        const int np = __popc(F);
                        if (firstp) s.tbl[__popc(F & lt)] = sk;
                        if ((int)lane >= np) s.tbl[lane] = INVALID_ID;
                        __syncwarp();
                        prod = INVALID_ID;
                        int l = (int)lane;
                        bool spare = false;
                        if (active) {
                            if (ar < np) prod = s.tbl[ar];
                            else { spare = true; l = (int)s.lane_of_rank[eq2_rank(ar, np, na)]; }
                        }
                        // ... spare lanes pick from served lane l's footprint (R-18 with |w|)
                        const int gx0 = __shfl_sync(FULL, x0, l), gy0 = __shfl_sync(FULL, y0, l);
                        const float gs = __shfl_sync(FULL, fs, l), gt = __shfl_sync(FULL, ft, l);
                        if (spare) {
                            const Foot16 g = footprint16(FILT, gx0, gy0, gs, gt, W, H);
                            float wsum = 0.0f;
                            float cw[16];
                            uint32_t cid[16];
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                const int rq = q >> 2, cq = q & 3;
                                const float mwq = __fmul_rn(sel4(g.mx, cq), sel4(g.my, rq));
                                const uint32_t id = (uint32_t)(g.ya + rq) * (uint32_t)W + (uint32_t)(g.xa + cq);
                                bool cand = rq < g.nr && cq < g.nc && mwq != 0.0f;
                                if (cand) {
                                    const int pos = lower_bound32(s.tbl, id);
                                    cand = !(pos < 32 && s.tbl[pos] == id);
                                }
                                cw[q] = cand ? fabsf(mwq) : 0.0f;
                                cid[q] = cand ? id : INVALID_ID;
                                if (cand) wsum = __fadd_rn(wsum, cw[q]);
                            }
                            if (wsum > 0.0f) {  // no candidate -> produce nothing
                                const float target = __fmul_rn(unit24(rnd.z), wsum);
                                float cum = 0.0f;
                                uint32_t pick = INVALID_ID, lastc = INVALID_ID;
#pragma unroll
                                for (int q = 0; q < 16; ++q) {
                                    if (cid[q] == INVALID_ID) continue;
                                    lastc = cid[q];
                                    cum = __fadd_rn(cum, cw[q]);
                                    if (pick == INVALID_ID && cum > target) pick = cid[q];
                                }
                                prod = pick != INVALID_ID ? pick : lastc;
                            }
                        }
                        __syncwarp();
                    }
                    // produce (one site), then every lane gathers the wave's produced set
                    float4 valf;
                    {
                        const uint32_t ty = prod != INVALID_ID ? prod / (uint32_t)W : 0u;
                        const uint32_t tx = prod != INVALID_ID ? prod - ty * (uint32_t)W : 0u;
                        if constexpr (TC) {
                            valf = mlp_decode_tc(a.tex, *tw, *tsc, prod != INVALID_ID, (int)tx, (int)ty, lane);
                            if (prod == INVALID_ID) valf = make_float4(0.f, 0.f, 0.f, 0.f);
                        } else {
                            Texel<FMT> val = Texel<FMT>::zero();
                            if (prod != INVALID_ID) val = produce(a.tex, mw, tx, ty);
                            valf = val.to_f4();
                        }
                    }
                    evals = (run_fb == FB_CPLUS) ? __popc(__ballot_sync(FULL, prod != INVALID_ID)) : na;
                    s.sorted[lane] = warp_sort32(prod != INVALID_ID ? ((prod << 5) | lane) : INVALID_ID);
                    s.xch[lane] = valf;   // this lane's produced value (fp32), read by lane index
                    __syncwarp();
                    // Eq. 1 over the known cells (R-23 evaluation order, R-28)
                    bool all_known = true;
                    int N = 0;
                    float Sw = 0.0f, Sp[4] = {0.f, 0.f, 0.f, 0.f};
                    Acc acc;
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int rq = q >> 2, cq = q & 3;
                        const float mwq = __fmul_rn(sel4(f.mx, cq), sel4(f.my, rq));
                        const bool need = active && rq < f.nr && cq < f.nc && mwq != 0.0f;
                        bool known = false;
                        int src = (int)lane;
                        if (need) {
                            const uint32_t id = (uint32_t)(f.ya + rq) * (uint32_t)W + (uint32_t)(f.xa + cq);
                            const int pos = lower_bound32(s.sorted, id << 5);
                            if (pos < 32) {
                                const uint32_t hit = s.sorted[pos];
                                if ((hit >> 5) == id) { known = true; src = (int)(hit & 31u); }
                            }
                        }
                        const float4 v = known ? s.xch[src] : make_float4(0.f, 0.f, 0.f, 0.f);
                        if (need && !known) all_known = false;
                        if (known) {
                            ++N;
                            Sw = __fadd_rn(Sw, mwq);
                            Sp[0] = __fadd_rn(Sp[0], v.x);
                            Sp[1] = __fadd_rn(Sp[1], v.y);
                            Sp[2] = __fadd_rn(Sp[2], v.z);
                            Sp[3] = __fadd_rn(Sp[3], v.w);
                        }
                        acc.add(mwq, v);
                    }
                    __syncwarp();
                    const float4 ac = acc.get();
                    const float rest = (all_known || N == 0) ? 0.0f : __fdividef(__fsub_rn(1.0f, Sw), (float)N);
                    color = make_float4(fmaf(rest, Sp[0], ac.x), fmaf(rest, Sp[1], ac.y), fmaf(rest, Sp[2], ac.z),
                                        fmaf(rest, Sp[3], ac.w));
                    if (N == 1 && !all_known) color = make_float4(Sp[0], Sp[1], Sp[2], Sp[3]);
                }
            }
            if (!active) color = make_float4(0.f, 0.f, 0.f, 0.f);
            if (inframe) st_stream_f4(a.out + pix, color);
            // ---- a8: record
            if (lane == 0) {
                const uint32_t ev = (uint32_t)evals;
                a.rec[widx] = (ev & 0xFFu) | ((uint32_t)(n & 0xFF) << 8) | ((uint32_t)na << 16) |
                              ((uint32_t)path << 22) | ((uint32_t)wave_mag << 25) | ((uint32_t)(na < 32) << 26) |
                              (((ev >> 8) & 7u) << 27);
            }
        }
    }
}

template <int FMT, int MODE>
static auto bicubic_kernel_for(int filt, bool box) {
    if constexpr (MODE == MODE_COLLAB)
        return filt == FILT_BSPLINE ? (box ? ctf_bicubic_kernel<FMT, MODE, FILT_BSPLINE, true>
                                           : ctf_bicubic_kernel<FMT, MODE, FILT_BSPLINE, false>)
                                    : (box ? ctf_bicubic_kernel<FMT, MODE, FILT_CATMULL_ROM, true>
                                           : ctf_bicubic_kernel<FMT, MODE, FILT_CATMULL_ROM, false>);
    else
        return filt == FILT_BSPLINE ? ctf_bicubic_kernel<FMT, MODE, FILT_BSPLINE, false>
                                    : ctf_bicubic_kernel<FMT, MODE, FILT_CATMULL_ROM, false>;
}

template <int FMT>
cudaError_t launch_bicubic(BArgs k, const typename WeightsOf<FMT>::type &mw, int mode, cudaStream_t stream) {
    const bool box = k.variant == BVAR_BOX;
    auto kern = mode == MODE_4TAP ? bicubic_kernel_for<FMT, MODE_4TAP>(k.filter, box)
              : mode == MODE_STF  ? bicubic_kernel_for<FMT, MODE_STF>(k.filter, box)
                                  : bicubic_kernel_for<FMT, MODE_COLLAB>(k.filter, box);
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    // latent MLP, collaborative: the tensor-core decoder's weights (per CTA) and scratch (per warp)
    const size_t dyn = (FMT == FMT_MLP && mode != MODE_4TAP && mode != MODE_STF)
                           ? sizeof(TcWeights) + kBWarps * sizeof(TcScratch) : 0;
    if (dyn > 0 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn)) != cudaSuccess)
        return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBWarps * 32, dyn);
    if (e != cudaSuccess) return e;
    const long long slots = (long long)sms * (per_sm > 0 ? per_sm : 1);
    long long ipw = ((long long)k.nchunks + slots * kBWarps * 4 - 1) / (slots * kBWarps * 4);
    ipw = ipw < 1 ? 1 : ipw > 4 ? 4 : ipw;
    k.ipw = (unsigned)ipw;
    long long grid = ((long long)k.nchunks + ipw * kBWarps - 1) / (ipw * kBWarps);
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kBWarps * 32, dyn, stream>>>(k, mw);
    return cudaGetLastError();
}

}  // namespace

#if CTF_TU_FMT == 1
bool bicubic_built() { return true; }
cudaError_t launch_bicubic_bc1(const LaunchArgs &a, cudaStream_t stream) {
#else
cudaError_t launch_bicubic_mlp(const LaunchArgs &a, cudaStream_t stream) {
#endif
    BArgs k;
    k.tex.W = a.W;
    k.tex.H = a.H;
    k.tex.bc1 = reinterpret_cast<const uint2 *>(a.tex_data);
    k.tex.latent = reinterpret_cast<const uint4 *>(a.tex_data);
    k.tex.mlp_dev = a.mlp;
    k.uv = reinterpret_cast<const float2 *>(a.uv);
    k.grad = reinterpret_cast<const uint2 *>(a.grad);
    k.out = reinterpret_cast<float4 *>(a.out);
    k.rec = a.rec;
    k.Wf = a.Wf;
    k.Hf = a.Hf;
    k.nwx = (a.Wf + 7) / 8;
    k.nwy = (a.Hf + 3) / 4;
    k.wpf = k.nwx * k.nwy;
    k.fpx = (unsigned)a.Wf * (unsigned)a.Hf;
    k.cpr = (k.nwx + kBChunk - 1) / kBChunk;
    k.cpf = k.cpr * k.nwy;
    k.nchunks = (unsigned)((long long)k.cpf * a.frames);
    k.ipw = 1;
    k.Wflt = (float)a.W;
    k.Hflt = (float)a.H;
    k.filter = a.filter;
    k.E = a.max_evals < 1 ? 1 : a.max_evals;
    k.fallback = a.fallback;
    k.variant = a.mode >= 4 ? a.mode - 3 : BVAR_LIST;
    k.flags = a.flags;
    k.frame_index = a.frame_index;
    k.row0 = a.row0;
    k.seed_lo = (uint32_t)a.seed;
    k.seed_hi = (uint32_t)(a.seed >> 32);
#if CTF_TU_FMT == 1
    return launch_bicubic<FMT_BC1>(k, NoWeights{}, a.mode, stream);
#else
    MlpWeights mw;
    const cudaError_t e = mlp_weights_by_value(a, stream, mw.v);
    if (e != cudaSuccess) return e;
    return launch_bicubic<FMT_MLP>(k, mw, a.mode, stream);
#endif
}

}  // namespace ctf
