// ctf_filter.cu — the collaborative texture filtering kernel (sm_100a).
//
// One 8x4-pixel wave = one warp.  Persistent grid: each warp walks
// waves w = gwarp, gwarp + S, ... over all frames of the batch (S = warps in the
// grid); the wave coordinates are advanced incrementally (no divisions).
// Per wave:
//   a1 load uv/grad (coalesced 64-B row segments), active mask A = ballot
//   a2 footprint: fx = u*W - 0.5, floor (magic-number, no F2I), clamp, weights
//   a3 collect: exact unique set U of the wave's footprint texels (List
//      semantics) in canonical ascending-id order (Mask h-order,
//      P:389-399).  Fast path: AABB by 4 redux.sync, then a row-major bitmask of
//      the AABB with power-of-two pitch (32/64/128 bits, specialised) OR-reduced
//      by redux.sync (WaveActiveBitOr) and popc ranks (h^-1).
//      Slow path: bitonic sort of the 128 footprint keys.
//   a4 decide: exact iff n <= popc(A)
//   a5 produce: active rank r < n produces texel U[r] (lane h(r,A))
//   a6 gather + blend: 4 __shfl_sync of packed RGBA8 (WaveReadLaneAt)
//   a7 fallback (n > a): STF / WC stand-in / C (Eq. 1) / C+ (Eq. 2); membership of
//      produced texels by AABB bitmask when it fits, else sorted keys
//   a8 per-wave record
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "ctf_device.cuh"
#include "ctf_internal.h"

namespace ctf {

constexpr int kWarps = 8;  // warps per CTA
#ifndef CTF_BC1_MINB
#define CTF_BC1_MINB 4  // BC1: resident CTAs per SM (64 registers)
#endif
#ifndef CTF_BC1_ROUNDS
#define CTF_BC1_ROUNDS 8  // BC1: target CTAs per resident CTA slot
#endif
#ifndef CTF_BC1_MAX_IPW
#define CTF_BC1_MAX_IPW 4  // BC1: at most this many work items per warp
#endif
#ifndef CTF_MLP_TC
#define CTF_MLP_TC 1  // latent-MLP COLLAB: tensor-core (3xFP16 mma.sync) wave decoder
#endif
#ifndef CTF_MLP_COLLAB_MINB
#define CTF_MLP_COLLAB_MINB 2  // latent-MLP COLLAB: resident CTAs per SM (register budget)
#endif

struct KArgs {
    TexArgs tex;
    const float2 *uv;
    const uint2 *grad;
    float4 *out;
    uint32_t *rec;
    uint32_t *dbg_pid, *dbg_sel, *dbg_unread;
    uint32_t *lcnt;                 // work-list counters [0] (fallback), [1] (general) when lists != NULL
    uint32_t *lists;                // optional work lists (BC1 COLLAB): fallback at [0], general at [nrec]
    unsigned nrec;                  // waves in the batch
    uint32_t wpf_m, nwx_m;          // magic multipliers: n / wpf, n / nwx (udiv_magic)
    int wpf_s, nwx_s;
    unsigned fpx;                   // pixels per frame (all pixel indices < 2^32, validated on the host)
    int Wf, Hf, nwx, nwy, wpf;
    int cpr, cpf;                   // work items (runs of `chunk` waves) per wave-row / per frame
    int chunk;                      // waves per work item (a run in one wave-row; <= 32, host-chosen)
    uint32_t cpr_m;                 // lean kernels: run j of a wave-row spans waves [j nwx / cpr, (j+1) nwx / cpr)
    int cpr_s;                      // (magic pair of the division by cpr, udiv_magic)
    unsigned nchunks;
    unsigned ipc;                   // work items per CTA (claimed dynamically by its warps)
    float Wflt, Hflt;
    int Wm1, Hm1;                   // texture W - 1, H - 1 (clamp-to-edge bounds)
    int fallback;
    int variant;                    // COLLAB kernel: VAR_LIST / VAR_BOX / VAR_MASK16 / VAR_MASK11
    uint32_t flags, frame_index, seed_lo, seed_hi;
    int row0;                       // frame row of buffer row 0 (strip sharding): RNG counter y = row0 + py
    uint32_t rk[2][10];             // Philox round keys of (seed_lo, seed_hi) (constant-bank operands)
};
enum { VAR_LIST = 0, VAR_BOX = 1, VAR_MASK16 = 2, VAR_MASK11 = 3 };

struct WarpSmem {
    uint32_t tbl[32];       // rank -> packed (y << 16 | x) of U[rank] (exact) / planned P (C+, sort path)
    uint32_t sorted[32];    // sorted (id << 5 | lane) of produced texels (fallback, sort path)
    uint8_t lane_of_rank[32];
    uint8_t lane_of_t[128]; // AABB position -> a lane that produced it (fallback, mask path)
    uint8_t rank_of[128];   // slow collect: (lane*4 + corner) -> rank
};

// n / d for n < 2^31 with a host-computed magic pair (m, s): s = floor(log2 d),
// m = ceil(2^(32+s) / d) (0 when d is a power of two), q = umulhi(n, m) >> s.  Exact: with
// m = 2^(32+s)/d + e (0 <= e < 1) the excess n e / 2^(32+s) stays below 1/d whenever
// n < 2^(32+s)/d, which holds for n < 2^31 because d < 2^(s+1).
__device__ __forceinline__ unsigned udiv_magic(unsigned n, uint32_t m, int s) { return (m ? __umulhi(n, m) : n) >> s; }
static inline void udiv_magic_host(unsigned d, uint32_t &m, int &s) {
    s = 31 - __builtin_clz(d);
    m = (d & (d - 1u)) == 0u ? 0u : (uint32_t)(((1ull << (32 + s)) + d - 1u) / d);
}

// Per-lane footprint of one pixel (a2).
struct Foot {
    int xa, xb, ya, yb;     // clamped texel columns / rows
    float s, t;             // fp32 fractional position (decides coordinates)
    float w[4];             // fp32 weights UL, UR, LL, LR, each product rounded once (R-3)
};

__device__ __forceinline__ void make_weights(Foot &f) {
    const float oms = __fsub_rn(1.0f, f.s), omt = __fsub_rn(1.0f, f.t);
    f.w[0] = __fmul_rn(oms, omt);
    f.w[1] = __fmul_rn(f.s, omt);
    f.w[2] = __fmul_rn(oms, f.t);
    f.w[3] = __fmul_rn(f.s, f.t);
}

// floor(v) for |v| < 2^22 without F2I/FRND: v + 1.5*2^23 rounded toward -inf lands
// on the integer grid, so its bits hold floor(v) and subtracting the magic is exact.
__device__ __forceinline__ int floor_split(float v, float &flo) {
    const float r = __fadd_rd(v, 12582912.0f);
    flo = __fsub_rn(r, 12582912.0f);
    return __float_as_int(r) - 0x4B400000;
}

__device__ __forceinline__ Foot footprint(float2 uv, const KArgs &a) {
    Foot f;
    // R-2: u, v clamped to [0, 1] (NaN -> 0), fx = fma(u, W, -0.5) (one rounding),
    // floor, exact s.  fx lies in [-0.5, W - 0.5], so x0 in [-1, W - 1]: only the
    // lower corner can fall below 0 and only the upper one above W - 1.
    const float fx = fmaf(__saturatef(uv.x), a.Wflt, -0.5f), fy = fmaf(__saturatef(uv.y), a.Hflt, -0.5f);
    float flx, fly;
    const int x0 = floor_split(fx, flx), y0 = floor_split(fy, fly);
    f.s = __fsub_rn(fx, flx);
    f.t = __fsub_rn(fy, fly);
    f.xa = max(x0, 0);
    f.xb = min(x0 + 1, a.Wm1);
    f.ya = max(y0, 0);
    f.yb = min(y0 + 1, a.Hm1);
    make_weights(f);
    return f;
}

// The same footprint with the x / y pairs in packed fp32 (FFMA2 / FADD2): every lane of a
// packed op is the scalar IEEE op, so the result equals footprint() bit for bit.
__device__ __forceinline__ uint64_t fadd2_rm(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ Foot footprint2(float2 uv, const KArgs &a) {
    Foot f;
    const uint64_t fxy = ffma2(f2pack(__saturatef(uv.x), __saturatef(uv.y)), f2pack(a.Wflt, a.Hflt),
                               f2pack(-0.5f, -0.5f));
    const uint64_t r = fadd2_rm(fxy, f2pack(12582912.0f, 12582912.0f));        // floor on the 2^23 grid
    const uint64_t st = ffma2(fadd2(r, f2pack(-12582912.0f, -12582912.0f)), f2pack(-1.0f, -1.0f), fxy);
    const float2 rr = f2unpack(r), stf = f2unpack(st);
    const int x0 = __float_as_int(rr.x) - 0x4B400000, y0 = __float_as_int(rr.y) - 0x4B400000;
    f.s = stf.x;
    f.t = stf.y;
    f.xa = max(x0, 0);
    f.xb = min(x0 + 1, a.Wm1);
    f.ya = max(y0, 0);
    f.yb = min(y0 + 1, a.Hm1);
    // {1 - s, 1 - t} in one FADD2 (one rounding each, as R-3), then the four products
    const float2 om = f2unpack(fsub2(f2pack(1.0f, 1.0f), st));
    f.w[0] = __fmul_rn(om.x, om.y);
    f.w[1] = __fmul_rn(f.s, om.y);
    f.w[2] = __fmul_rn(om.x, f.t);
    f.w[3] = __fmul_rn(f.s, f.t);
    return f;
}

__device__ __forceinline__ int corner_x(const Foot &f, int k) { return (k & 1) ? f.xb : f.xa; }
__device__ __forceinline__ int corner_y(const Foot &f, int k) { return (k & 2) ? f.yb : f.ya; }
__device__ __forceinline__ uint32_t corner_id(const Foot &f, int k, int W) {
    return (uint32_t)(corner_y(f, k) * W + corner_x(f, k));
}

// Exact bilinear of 4 gathered texels (c8).  The same code runs in 4TAP and in
// COLLAB-exact, so the two are bit-identical on exact waves.
// Texel values as fp32 in [0, 1] (BC1: v * fl(1/255), R-9), then the
// FFMA2 chain of blend4f.
template <int FMT>
__device__ __forceinline__ float4 blend4(const Texel<FMT> (&p)[4], const float (&w)[4]) {
    const float4 v[4] = {p[0].to_f4(), p[1].to_f4(), p[2].to_f4(), p[3].to_f4()};
    return blend4f(v, w);
}

template <int FMT>
__device__ __forceinline__ float4 scaled(const Texel<FMT> &p) { return p.to_f4(); }

// Eq. 2 generalised to a active lanes (R-18 iv), round half up.
// floor(num / den) for 0 <= num < 2^11, 0 < den <= 62 as trunc((num + 1/2) / den) with the
// approximate division (MUFU.RCP + FMUL, relative error < 2^-21): the fractional part of
// (num + 1/2) / den lies in [1/(2 den), 1 - 1/(2 den)], a margin of >= 1/124 against an
// absolute error < 32 * 2^-21, so the result is the exact integer quotient
// (tests/test_kernel_arith.py checks the margin for every (j, np, na)).
__device__ __forceinline__ int eq2_lane_rank(int j, int np, int na) {
    if (np >= na - 1) return 0;
    const int num = 2 * (na - 1) * (j - np) + (na - 1 - np);
    const int den = 2 * (na - 1 - np);
    return __float2int_rz(__fdividef((float)num + 0.5f, (float)den));
}

// STF corner (R-12): dx = (u0 < s), dy = (u1 < t).
__device__ __forceinline__ int stf_corner(const Foot &f, uint4 r) {
    return (unit24(r.x) < f.s ? 1 : 0) + (unit24(r.y) < f.t ? 2 : 0);
}

// ------------------------------------------------------------------ AABB bitmask
// Wave bounding-box origin (min corner, 2 redux.sync) and a bitmask window of width
// 2^lgP anchored there: bit t = (y - miny) * 2^lgP + (x - minx).  The window shape is
// the first of 8x4, 4x8 (32 bits), 8x8 (64), 16x8, 8x16, 32x4 (128) that holds every
// active footprint (one vote each); K = words, 0 = does not fit (sort path).
struct Box {
    int minx, miny, lgP, K;
    bool fits;
};

__device__ __forceinline__ Box wave_box(const Foot &f, bool active) {
    Box b;
    b.minx = __reduce_min_sync(FULL, active ? f.xa : INT_MAX);
    b.miny = __reduce_min_sync(FULL, active ? f.ya : INT_MAX);
    const unsigned dx = (unsigned)(f.xb - b.minx), dy = (unsigned)(f.yb - b.miny);
    if (__all_sync(FULL, !active || (dx < 8u && dy < 4u))) { b.lgP = 3; b.K = 1; }
    else if (__all_sync(FULL, !active || (dx < 4u && dy < 8u))) { b.lgP = 2; b.K = 1; }
    else if (__all_sync(FULL, !active || (dx < 8u && dy < 8u))) { b.lgP = 3; b.K = 2; }
    else if (__all_sync(FULL, !active || (dx < 16u && dy < 8u))) { b.lgP = 4; b.K = 4; }
    else if (__all_sync(FULL, !active || (dx < 8u && dy < 16u))) { b.lgP = 3; b.K = 4; }
    else if (__all_sync(FULL, !active || (dx < 32u && dy < 4u))) { b.lgP = 5; b.K = 4; }
    else { b.lgP = 0; b.K = 0; }
    b.fits = b.K != 0;
    return b;
}
__device__ __forceinline__ uint32_t box_t(const Box &b, int x, int y) {
    return ((uint32_t)(y - b.miny) << b.lgP) + (uint32_t)(x - b.minx);
}
__device__ __forceinline__ int box_x(const Box &b, uint32_t t) { return b.minx + (int)(t & ((1u << b.lgP) - 1u)); }
__device__ __forceinline__ int box_y(const Box &b, uint32_t t) { return b.miny + (int)(t >> b.lgP); }

// K-word (K*32-bit) wave mask, OR-reduced across the warp.
template <int K>
struct WMask {
    uint32_t w[K];
    int pre[K];
    int n;
    __device__ __forceinline__ uint32_t word(uint32_t k) const {
        if constexpr (K == 1) return w[0];
        else if constexpr (K == 2) return k == 0 ? w[0] : w[1];
        else return k == 0 ? w[0] : k == 1 ? w[1] : k == 2 ? w[2] : w[3];
    }
    __device__ __forceinline__ int prefix(uint32_t k) const {
        if constexpr (K == 1) return 0;
        else if constexpr (K == 2) return k == 0 ? 0 : pre[1];
        else return k == 0 ? 0 : k == 1 ? pre[1] : k == 2 ? pre[2] : pre[3];
    }
    __device__ __forceinline__ void finish() {
        n = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) { pre[k] = n; n += __popc(w[k]); }
    }
    // OR of a 2-bit pattern at t0 and t2 (a lane's 2x2 footprint; rows never straddle words)
    __device__ __forceinline__ void reduce_2x2(uint32_t t0, uint32_t t2, uint32_t pat, bool on) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            uint32_t m = 0u;
            if (on) {
                if (K == 1 || (t0 >> 5) == (uint32_t)k) m |= pat << (t0 & 31u);
                if (K == 1 || (t2 >> 5) == (uint32_t)k) m |= pat << (t2 & 31u);
            }
            w[k] = __reduce_or_sync(FULL, m);
        }
        finish();
    }
    __device__ __forceinline__ void reduce_bit(uint32_t t, bool on) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            w[k] = __reduce_or_sync(FULL, (on && (t >> 5) == (uint32_t)k) ? (1u << (t & 31u)) : 0u);
        finish();
    }
    __device__ __forceinline__ int rank(uint32_t t) const {
        return prefix(t >> 5) + __popc(word(t >> 5) & ((1u << (t & 31u)) - 1u));
    }
    __device__ __forceinline__ bool test(uint32_t t) const { return (word(t >> 5) >> (t & 31u)) & 1u; }
    // lane j owns bit j of every word: write rank -> bit position t for ranks < 32
    __device__ __forceinline__ void push(uint32_t *tbl, unsigned lane, unsigned lt) const {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if ((w[k] >> lane) & 1u) {
                const int r = pre[k] + __popc(w[k] & lt);
                if (r < 32) tbl[r] = ((uint32_t)k << 5) | lane;
            }
        }
    }
};

// ------------------------------------------------------------- fallback gather
// distinct corners in first-occurrence order + merged fp32 weights; dup[k] = first corner
// holding the same texel (texel identity by packed (y << 16 | x)).
__device__ __forceinline__ void distinct_corners(const Foot &f, bool (&first)[4], float (&dw)[4], int (&dup)[4]) {
    const uint32_t key[4] = {((uint32_t)f.ya << 16) | (uint32_t)f.xa, ((uint32_t)f.ya << 16) | (uint32_t)f.xb,
                             ((uint32_t)f.yb << 16) | (uint32_t)f.xa, ((uint32_t)f.yb << 16) | (uint32_t)f.xb};
#pragma unroll
    for (int k = 0; k < 4; ++k) { first[k] = true; dw[k] = f.w[k]; dup[k] = k; }
#pragma unroll
    for (int k = 1; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < k; ++j)
            if (first[j] && first[k] && key[j] == key[k]) {
                first[k] = false;
                dup[k] = j;
                dw[j] = __fadd_rn(dw[j], f.w[k]);
            }
}

// Eq. 1 / WC combine from the gathered values of the lane's distinct corners (c14-c16).
__device__ __forceinline__ float4 combine_eq1f(const Foot &f, const bool (&first)[4], const float (&dw)[4],
                                               const bool (&known)[4], const int (&dup)[4], const float4 (&pv)[4],
                                               bool wc) {
    // Branch-free over the lane's cases (R-23).  Every nonzero-weight texel known -> blend4
    // over the corners, i.e. exact bilinear bit for bit (c8).  Otherwise C / C+
    // evaluate Eq. 1 as one blend4 with per-corner coefficients w_k + rest (combine_eq1_coef;
    // N = 1 gives (dw + (1 - dw)) p = p to fp32 rounding), which agrees with the oracle's
    // fmaf chain to fp32 rounding; WC (R-16) renormalises, N = 1 -> that texel exactly.
    bool all_known = true;
    int N = 0;
    float Sw = 0.f, Sp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!first[k] || dw[k] == 0.0f) continue;
        if (!known[k]) { all_known = false; continue; }
        ++N;
        Sw += dw[k];
        Sp[0] += pv[k].x; Sp[1] += pv[k].y; Sp[2] += pv[k].z; Sp[3] += pv[k].w;
    }
    float4 q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int d = dup[k];
        const float4 src = d == 0 ? pv[0] : d == 1 ? pv[1] : d == 2 ? pv[2] : pv[3];
        const bool kd = d == 0 ? known[0] : d == 1 ? known[1] : d == 2 ? known[2] : known[3];
        q[k] = kd ? src : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float4 bl = blend4f(q, f.w);  // sum over the known corners of w_k p_k
    const bool one = N == 1 && !all_known;
    float c[4];
    if (wc) {  // WC stand-in (R-16): weights renormalised over the known texels
        float Swp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!first[k] || dw[k] == 0.0f || !known[k]) continue;
            Swp[0] = fmaf(dw[k], pv[k].x, Swp[0]);
            Swp[1] = fmaf(dw[k], pv[k].y, Swp[1]);
            Swp[2] = fmaf(dw[k], pv[k].z, Swp[2]);
            Swp[3] = fmaf(dw[k], pv[k].w, Swp[3]);
        }
        const float r = 1.0f / Sw;
        c[0] = all_known ? bl.x : Swp[0] * r;
        c[1] = all_known ? bl.y : Swp[1] * r;
        c[2] = all_known ? bl.z : Swp[2] * r;
        c[3] = all_known ? bl.w : Swp[3] * r;
    } else {  // Eq. 1: the coefficient blend of combine_eq1_coef (same operations in
              // the same order, so the general and wide-window paths agree bit for bit)
        const float rest = (all_known || N == 0) ? 0.0f : __fdividef(1.0f - Sw, (float)N);
        float cf[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int d = dup[k];
            const bool kd = d == 0 ? known[0] : d == 1 ? known[1] : d == 2 ? known[2] : known[3];
            const bool kn = first[k] && dw[k] != 0.0f && known[k];
            cf[k] = __fadd_rn(kd ? f.w[k] : 0.0f, kn ? rest : 0.0f);
        }
        return blend4f(q, cf);
    }
    if (one) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) c[ch] = Sp[ch];
    }
    return make_float4(c[0], c[1], c[2], c[3]);
}
template <int FMT>
__device__ __forceinline__ float4 combine_eq1(const Foot &f, const bool (&first)[4], const float (&dw)[4],
                                              const bool (&known)[4], const int (&dup)[4], const Texel<FMT> (&p)[4],
                                              bool wc) {
    const float4 pv[4] = {p[0].to_f4(), p[1].to_f4(), p[2].to_f4(), p[3].to_f4()};   // texel values in [0, 1]
    return combine_eq1f(f, first, dw, known, dup, pv, wc);
}

// Gather via sorted (id << 5 | lane) keys + binary search (any AABB size).
template <int FMT>
__device__ __forceinline__ float4 gather_sorted(const Foot &f, bool active, uint32_t prod, const Texel<FMT> &val,
                                                bool wc, WarpSmem &s, int W) {
    const unsigned lane = lane_id();
    const uint32_t key = (active && prod != INVALID_ID) ? ((prod << 5) | lane) : INVALID_ID;
    s.sorted[lane] = warp_sort32(key);
    __syncwarp();
    bool first[4], known[4];
    float dw[4];
    int dup[4], src[4];
    distinct_corners(f, first, dw, dup);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        known[k] = false;
        src[k] = (int)lane;
        if (active && first[k] && dw[k] != 0.0f) {
            const uint32_t id = corner_id(f, k, W);
            const int pos = lower_bound32(s.sorted, id << 5);
            if (pos < 32) {
                const uint32_t hit = s.sorted[pos];
                if ((hit >> 5) == id) { known[k] = true; src[k] = (int)(hit & 31u); }
            }
        }
    }
    Texel<FMT> p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = Texel<FMT>::shfl(val, src[k]);
    __syncwarp();
    if (!active) return make_float4(0.f, 0.f, 0.f, 0.f);
    return combine_eq1<FMT>(f, first, dw, known, dup, p, wc);
}

// Gather via the AABB bitmask of produced texels + a position -> lane table.
template <int FMT>
__device__ __forceinline__ float4 gather_mask(const Foot &f, const Box &b, bool active, bool produced,
                                              uint32_t prod_t, const Texel<FMT> &val, bool wc, WarpSmem &s) {
    const unsigned lane = lane_id();
    WMask<4> D;
    D.reduce_bit(prod_t, active && produced);
    // several lanes may produce the same texel (STF, C+ extras): __match_any_sync groups
    // them and only the lowest lane of each group publishes itself as the source of t
    const unsigned peers = __match_any_sync(FULL, (active && produced) ? prod_t : 0xFFFFFFFFu);
    if (active && produced && (unsigned)(__ffs(peers) - 1) == lane) s.lane_of_t[prod_t] = (uint8_t)lane;
    __syncwarp();
    bool first[4], known[4];
    float dw[4];
    int dup[4], src[4];
    distinct_corners(f, first, dw, dup);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        known[k] = false;
        src[k] = (int)lane;
        if (active && first[k] && dw[k] != 0.0f) {
            const uint32_t t = box_t(b, corner_x(f, k), corner_y(f, k));
            if (D.test(t)) { known[k] = true; src[k] = s.lane_of_t[t]; }
        }
    }
    Texel<FMT> p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = Texel<FMT>::shfl(val, src[k]);
    __syncwarp();
    if (!active) return make_float4(0.f, 0.f, 0.f, 0.f);
    return combine_eq1<FMT>(f, first, dw, known, dup, p, wc);
}

// ------------------------------------------------------------------ fallbacks
// A fallback runs in two phases around the kernel's single texel-production site:
//   fb_plan   decides which texel (if any) this lane produces (STF choice, C+ plan
//             and Eq. 2 spare-lane picks), and
//   fb_finish gathers the produced values of the wave and combines them (Eq. 1 / WC),
// so no fallback code needs the texture decoder (or the MLP weights).
struct Plan {
    bool produced;
    int qx, qy;          // texel this lane produces
    int ksel;            // STF corner of this lane's own pixel
    uint32_t selbits;
};

// C+ spare lane: candidate pick from served lane l's footprint g (R-18 v): distinct
// nonzero-weight texels not in the plan, chosen with probability ~ merged weight.
template <typename Planned>
__device__ __forceinline__ int cplus_pick(const Foot &g, float u2, Planned planned) {
    bool first[4];
    float cw[4];
    int dup[4];
    distinct_corners(g, first, cw, dup);
    bool cand[4];
    float wsum = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cand[k] = first[k] && cw[k] != 0.0f && !planned(corner_x(g, k), corner_y(g, k));
        if (cand[k]) wsum = __fadd_rn(wsum, cw[k]);
    }
    if (!(cand[0] || cand[1] || cand[2] || cand[3])) return -1;
    const float target = __fmul_rn(u2, wsum);
    float cum = 0.0f;
    int pick = -1, lastc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!cand[k]) continue;
        lastc = k;
        cum = __fadd_rn(cum, cw[k]);
        if (pick < 0 && cum > target) pick = k;
    }
    return pick < 0 ? lastc : pick;
}

__device__ __forceinline__ Plan fb_plan_impl(int fb, const Foot &f, const Box &b, bool active, unsigned A, int na,
                                              int px, int py, uint32_t frame, uint32_t seed_lo, uint32_t seed_hi,
                                              int W, WarpSmem &s) {
    const unsigned lane = lane_id();
    const unsigned lt = lanemask_lt();
    Plan pl;
    const uint4 rr = philox4x32_10(make_uint4((uint32_t)px, (uint32_t)py, frame, 0u), seed_lo, seed_hi);
    pl.ksel = stf_corner(f, rr);
    pl.selbits = active ? (uint32_t)pl.ksel : 0u;
    pl.qx = corner_x(f, pl.ksel);
    pl.qy = corner_y(f, pl.ksel);
    pl.produced = active;
    if (fb != FB_CPLUS) return pl;  // STF, WC, C: every lane produces its STF texel

    // ---- C+ (P:485-518): (1) planned STF texels, deduplicated and ranked ascending
    pl.produced = false;
    const int ar = __popc(A & lt);
    if (active) s.lane_of_rank[ar] = (uint8_t)lane;
    int np;
    WMask<4> P;
    if (b.fits) {
        P.reduce_bit(box_t(b, pl.qx, pl.qy), active);   // one bit per lane
        np = P.n;
        P.push(s.tbl, lane, lt);
    } else {
        const uint32_t pid = (uint32_t)(pl.qy * W + pl.qx);
        const uint32_t sk = warp_sort32(active ? ((pid << 5) | lane) : INVALID_ID);
        const uint32_t skp = __shfl_up_sync(FULL, sk, 1);
        const bool firstp = sk != INVALID_ID && (lane == 0 || (sk >> 5) != (skp >> 5));
        const unsigned F = __ballot_sync(FULL, firstp);
        np = __popc(F);
        if (firstp) s.tbl[__popc(F & lt)] = sk >> 5;   // sorted planned ids
        if ((int)lane >= np) s.tbl[lane] = INVALID_ID;
    }
    __syncwarp();
    // (2) active ranks < n_p produce the planned texels; (3) the rest are spare lanes (Eq. 2)
    bool spare = false;
    int l = (int)lane;
    if (active) {
        if (ar < np) {
            const uint32_t e = s.tbl[ar];
            if (b.fits) { pl.qx = box_x(b, e); pl.qy = box_y(b, e); }
            else { pl.qy = (int)(e / (uint32_t)W); pl.qx = (int)(e - (uint32_t)pl.qy * (uint32_t)W); }
            pl.produced = true;
        } else {
            spare = true;
            l = (int)s.lane_of_rank[eq2_lane_rank(ar, np, na)];
            pl.selbits |= (1u << 5) | ((uint32_t)l << 8);
        }
    }
    Foot g;
    g.xa = __shfl_sync(FULL, f.xa, l);
    g.xb = __shfl_sync(FULL, f.xb, l);
    g.ya = __shfl_sync(FULL, f.ya, l);
    g.yb = __shfl_sync(FULL, f.yb, l);
    g.s = __shfl_sync(FULL, f.s, l);
    g.t = __shfl_sync(FULL, f.t, l);
    if (spare) {
        make_weights(g);
        int pick;
        if (b.fits) {
            pick = cplus_pick(g, unit24(rr.z), [&](int x, int y) { return P.test(box_t(b, x, y)); });
        } else {
            pick = cplus_pick(g, unit24(rr.z), [&](int x, int y) {
                const uint32_t id = (uint32_t)(y * W + x);
                const int pos = lower_bound32(s.tbl, id);
                return pos < 32 && s.tbl[pos] == id;
            });
        }
        if (pick >= 0) {
            pl.qx = corner_x(g, pick);
            pl.qy = corner_y(g, pick);
            pl.produced = true;
            pl.selbits |= ((uint32_t)pick << 2) | (1u << 4);
        }
    }
    __syncwarp();
    return pl;
}

struct Finished {
    float4 color;
    int evals;
};

// (4) every lane filters with the produced texels of the wave: one-tap (STF), the WC
// stand-in, or Eq. 1 (C, C+)
template <int FMT>
__device__ __forceinline__ Finished fb_finish_impl(int fb, const Foot &f, const Box &b, bool active, int na,
                                                   const Plan &pl, const Texel<FMT> &val, int W, WarpSmem &s) {
    Finished o;
    if (fb == FB_STF) {
        o.evals = na;
        o.color = active ? scaled<FMT>(val) : make_float4(0.f, 0.f, 0.f, 0.f);
        return o;
    }
    o.evals = (fb == FB_CPLUS) ? __popc(__ballot_sync(FULL, active && pl.produced)) : na;
    const bool wc = fb == FB_WC;
    if (b.fits)
        o.color = gather_mask<FMT>(f, b, active, pl.produced, box_t(b, pl.qx, pl.qy), val, wc, s);
    else
        o.color = gather_sorted<FMT>(f, active, pl.produced ? (uint32_t)(pl.qy * W + pl.qx) : INVALID_ID, val, wc,
                                     s, W);
    return o;
}

// Out-of-line entry points.  Latent-MLP: plan and finish are separate calls so the
// kernel keeps ONE inline copy of the 1.5k-FMA decoder (its weights are kernel
// parameters).  BC1: plan + decode + finish in one out-of-line call (cheap decoder,
// smaller hot loop).
static __device__ __noinline__ Plan fb_plan(int fb, const Foot f, const Box b, bool active, unsigned A, int na, int px,
                                            int py, uint32_t frame, uint32_t seed_lo, uint32_t seed_hi, int W,
                                            WarpSmem &s) {
    return fb_plan_impl(fb, f, b, active, A, na, px, py, frame, seed_lo, seed_hi, W, s);
}
template <int FMT>
static __device__ __noinline__ Finished fb_finish(int fb, const Foot f, const Box b, bool active, int na, const Plan pl,
                                                  const Texel<FMT> val, int W, WarpSmem &s) {
    return fb_finish_impl<FMT>(fb, f, b, active, na, pl, val, W, s);
}
struct FbAll {
    Finished fin;
    uint32_t prod, selbits;
};
static __device__ __noinline__ FbAll fb_all_bc1(int fb, const Foot f, const Box b, bool active, unsigned A, int na,
                                                int px, int py, uint32_t frame, const KArgs &a, WarpSmem &s) {
    const int W = a.tex.W;
    const Plan pl = fb_plan_impl(fb, f, b, active, A, na, px, py, frame, a.seed_lo, a.seed_hi, W, s);
    Texel<FMT_BC1> val = Texel<FMT_BC1>::zero();
    FbAll r;
    r.prod = INVALID_ID;
    r.selbits = pl.selbits;
    if (pl.produced) {
        val = produce(a.tex, NoWeights{}, pl.qx, pl.qy);
        r.prod = (uint32_t)(pl.qy * W + pl.qx);
    }
    r.fin = fb_finish_impl<FMT_BC1>(fb, f, b, active, na, pl, val, W, s);
    return r;
}

// --------------------------------------------------------------- exact collect
template <int K>
__device__ __forceinline__ int collect_mask(const Foot &f, const Box &b, bool active, int (&rho)[4], WarpSmem &s,
                                            unsigned lane) {
    const uint32_t t0 = box_t(b, f.xa, f.ya);
    const uint32_t t2 = t0 + ((uint32_t)(f.yb - f.ya) << b.lgP);
    const uint32_t dxs = (uint32_t)(f.xb - f.xa);
    WMask<K> B;
    B.reduce_2x2(t0, t2, 1u | (dxs << 1), active);
    rho[0] = B.rank(t0);
    rho[1] = rho[0] + (int)dxs;
    rho[2] = B.rank(t2);
    rho[3] = rho[2] + (int)dxs;
    if (B.n <= 32) B.push(s.tbl, lane, lanemask_lt());
    return B.n;
}

struct Collected {
    int n;
    int rho[4];
};

static __device__ __noinline__ Collected collect_sort(const Foot f, bool active, WarpSmem &s, unsigned lane, int W) {
    Collected c;
    uint32_t key[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        key[k] = active ? ((corner_id(f, k, W) << 7) | (lane << 2) | (uint32_t)k) : INVALID_ID;
    warp_sort128(key);
    const uint32_t prev = __shfl_up_sync(FULL, key[3], 1);
    int fl[4];
    fl[0] = key[0] != INVALID_ID && (lane == 0 || (key[0] >> 7) != (prev >> 7));
#pragma unroll
    for (int k = 1; k < 4; ++k) fl[k] = key[k] != INVALID_ID && (key[k] >> 7) != (key[k - 1] >> 7);
    const int cnt = fl[0] + fl[1] + fl[2] + fl[3];
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(FULL, incl, d);
        if ((int)lane >= d) incl += o;
    }
    c.n = __shfl_sync(FULL, incl, 31);
    int run = incl - cnt;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        run += fl[k];
        if (key[k] != INVALID_ID) {
            const int r = run - 1;
            s.rank_of[key[k] & 127u] = (uint8_t)r;
            if (fl[k] && r < 32) {
                const uint32_t id = key[k] >> 7;
                const uint32_t y = id / (uint32_t)W;
                s.tbl[r] = (y << 16) | (id - y * (uint32_t)W);
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) c.rho[k] = active ? (int)s.rank_of[lane * 4 + k] : 0;
    return c;
}

// ------------------------------------------------ wave-batched latent-MLP decode
// The n unique texels of an exact wave are decoded TOGETHER: lane j owns hidden unit j
// (its rows of W1 and W2 live in registers for the whole kernel) and loops over the n
// texels; the producer of texel r only computes its 12 inputs and the 4 outputs.  Per
// wave: ~62 instructions per texel + ~190 fixed, instead of the full 1.5k-FMA decoder on
// every lane (SIMT).  Each output is the same sequence of fp32 operations as mlp_decode,
// so the texels are bit-identical (P:855-869 split decode across lanes).
struct MlpBatchSmem {
    float4 in[32][3];    // texel r's 12 inputs (rows >= n are never consumed)
    float h1[4][32];     // layer-1 activations of the 4 texels in flight
    float h2[32][36];    // layer-2 activations per texel (row stride 36: conflict-free LDS.128)
};

struct MlpLaneWeights {
    float w1[12], w2[32], b1, b2;   // row `lane` of W1 / W2 and its biases (ABI layout)
};

__device__ __forceinline__ void load_lane_weights(const float *__restrict__ m, unsigned lane, MlpLaneWeights &lw) {
#pragma unroll
    for (int i = 0; i < 12; ++i) lw.w1[i] = __ldg(m + lane * 12 + i);
    lw.b1 = __ldg(m + 384 + lane);
#pragma unroll
    for (int k = 0; k < 32; ++k) lw.w2[k] = __ldg(m + 416 + lane * 32 + k);
    lw.b2 = __ldg(m + 1440 + lane);
}

// Texels are processed 4 at a time so every lane runs 4 independent FMA chains.
__device__ __forceinline__ float4 mlp_decode_batched(const TexArgs &t, const MlpWeights &mw, MlpBatchSmem &ms,
                                                     const MlpLaneWeights &lw, bool producer, int r, int qx, int qy,
                                                     int n, unsigned lane) {
    if (producer) {
        float in[12];
        mlp_features(t, qx, qy, in);
        ms.in[r][0] = make_float4(in[0], in[1], in[2], in[3]);
        ms.in[r][1] = make_float4(in[4], in[5], in[6], in[7]);
        ms.in[r][2] = make_float4(in[8], in[9], in[10], in[11]);
    }
    __syncwarp();
    for (int t0 = 0; t0 < n; t0 += 4) {
        // layer 1: lane = hidden unit, 4 texels
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int tq = min(t0 + q, 31);
            const float4 i0 = ms.in[tq][0], i1 = ms.in[tq][1], i2 = ms.in[tq][2];
            float h = lw.b1;
            h = fmaf(lw.w1[0], i0.x, h); h = fmaf(lw.w1[1], i0.y, h); h = fmaf(lw.w1[2], i0.z, h);
            h = fmaf(lw.w1[3], i0.w, h); h = fmaf(lw.w1[4], i1.x, h); h = fmaf(lw.w1[5], i1.y, h);
            h = fmaf(lw.w1[6], i1.z, h); h = fmaf(lw.w1[7], i1.w, h); h = fmaf(lw.w1[8], i2.x, h);
            h = fmaf(lw.w1[9], i2.y, h); h = fmaf(lw.w1[10], i2.z, h); h = fmaf(lw.w1[11], i2.w, h);
            ms.h1[q][lane] = fmaxf(h, 0.f);
        }
        __syncwarp();
        // layer 2: lane = hidden unit, 4 texels, k ascending (same order as mlp_decode)
        float acc[4] = {lw.b2, lw.b2, lw.b2, lw.b2};
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 hv = reinterpret_cast<const float4 *>(ms.h1[q])[k4];
                acc[q] = fmaf(lw.w2[4 * k4 + 0], hv.x, acc[q]);
                acc[q] = fmaf(lw.w2[4 * k4 + 1], hv.y, acc[q]);
                acc[q] = fmaf(lw.w2[4 * k4 + 2], hv.z, acc[q]);
                acc[q] = fmaf(lw.w2[4 * k4 + 3], hv.w, acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (t0 + q < 32) ms.h2[t0 + q][lane] = fmaxf(acc[q], 0.f);
        __syncwarp();
    }
    // layer 3: the producer of texel r forms its 4 outputs (weights warp-uniform)
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (producer) {
        const float *W3T = mw.v + 1472, *b3 = mw.v + 1600;   // kernel layout: W3T[j][c], b3[c]
        float oc[4] = {b3[0], b3[1], b3[2], b3[3]};
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
            const float4 hv = *reinterpret_cast<const float4 *>(&ms.h2[r][4 * j4]);
            const float hj[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int c = 0; c < 4; ++c) oc[c] = fmaf(W3T[(4 * j4 + jj) * 4 + c], hj[jj], oc[c]);
        }
        o = make_float4(fminf(fmaxf(oc[0], 0.f), 1.f), fminf(fmaxf(oc[1], 0.f), 1.f), fminf(fmaxf(oc[2], 0.f), 1.f),
                        fminf(fmaxf(oc[3], 0.f), 1.f));
    }
    return o;
}

#include "ctf_mlp_tc.cuh"

// ----------------------------------------------------------------------- kernel
#ifndef CTF_CHUNK
#define CTF_CHUNK 16
#endif
constexpr int kChunk = CTF_CHUNK;  // waves per work item: a run of consecutive waves in one wave-row (<= 32)
static_assert(kChunk >= 1 && kChunk <= 32, "a run's records are buffered one per lane");

struct MlpCtx {  // latent-MLP COLLAB decoder state (unused by BC1)
    TcWeights *tw;
    TcScratch *tsc;
    MlpLaneWeights *lw;
    unsigned char *dyn;
    unsigned warp;
};

struct WaveOut {
    float4 color;
    uint32_t rec, prod, selbits;
};

// One live wave (A != 0) through the general path: every mode, Box / Mask variant,
// window size, partial wave and fallback.  The BC1 COLLAB List kernel below sends only
// its rare waves here (out of line).
template <int FMT, int MODE, bool DBG>
__device__ __forceinline__ WaveOut wave_general(const KArgs &a, const typename WeightsOf<FMT>::type &mw, WarpSmem &s,
                                                const MlpCtx &mc, float2 uv, uint2 gr, bool active, unsigned A,
                                                int na, int px, int py, uint32_t frame) {
    const unsigned lane = lane_id();
    const unsigned lt = lanemask_lt();
    constexpr bool kBatchMlp = FMT == FMT_MLP && MODE == MODE_COLLAB;
    (void)mc;
    (void)kBatchMlp;
    // Partial wave: inactive lanes borrow the first active lane's inputs, so the
    // wave-wide reductions below need no per-lane predicates (a duplicate footprint
    // changes no min, max, OR or unique set).  Their outputs are discarded.
    float2 uvm = uv;
    uint2 grm = gr;
    if (A != FULL) {
        const int leader = __ffs(A) - 1;
        const float lu = __shfl_sync(FULL, uv.x, leader), lv = __shfl_sync(FULL, uv.y, leader);
        const unsigned g0 = __shfl_sync(FULL, gr.x, leader), g1 = __shfl_sync(FULL, gr.y, leader);
        if (!active) {
            uvm = make_float2(lu, lv);
            grm = make_uint2(g0, g1);
        }
    }
    bool mag_lane = true;
    if (a.grad) {
        // R-20: squares of fp16 values are exact in fp32, so fma(g0, g0, g1*g1)
        // rounds once exactly like the fp32 sum of the two products
        const float rx = fma_f32_f16((unsigned short)(grm.x & 0xffffu), (unsigned short)(grm.x & 0xffffu),
                                     fma_f32_f16((unsigned short)(grm.x >> 16), (unsigned short)(grm.x >> 16), 0.0f));
        const float ry = fma_f32_f16((unsigned short)(grm.y & 0xffffu), (unsigned short)(grm.y & 0xffffu),
                                     fma_f32_f16((unsigned short)(grm.y >> 16), (unsigned short)(grm.y >> 16), 0.0f));
        mag_lane = rx <= 1.0f && ry <= 1.0f;  // max(rx, ry) <= 1
    }
    const bool wave_mag = a.grad != nullptr && __all_sync(FULL, mag_lane);
    const uint32_t rec_base = ((uint32_t)na << 16) | ((uint32_t)wave_mag << 25) | ((uint32_t)(na < 32) << 26);

    // ---- a2: footprint
    const Foot f = footprint(uvm, a);

    uint32_t prod = INVALID_ID, selbits = 0u, rec;
    float4 color = make_float4(0.f, 0.f, 0.f, 0.f);

    if constexpr (MODE == MODE_4TAP) {
        rec = rec_base | (0xFFu << 8) | ((uint32_t)PATH_4TAP << 22) | (uint32_t)((4 * na) & 0xFF);
        if (active) {
            if constexpr (FMT == FMT_BC1) {
                Texel<FMT> p[4];
                p[0] = produce(a.tex, mw, f.xa, f.ya);
                p[1] = produce(a.tex, mw, f.xb, f.ya);
                p[2] = produce(a.tex, mw, f.xa, f.yb);
                p[3] = produce(a.tex, mw, f.xb, f.yb);
                color = blend4<FMT>(p, f.w);
            } else {
                // one decode at a time (no interleaving of four MLPs); same op order as blend4
                float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
                for (int k = 0; k < 4; ++k) {
                    const float4 v = produce(a.tex, mw, corner_x(f, k), corner_y(f, k)).v;
                    const float wk = (k == 0 ? f.w[0] : k == 1 ? f.w[1] : k == 2 ? f.w[2] : f.w[3]);
                    if (k == 0) {
                        c[0] = wk * v.x; c[1] = wk * v.y; c[2] = wk * v.z; c[3] = wk * v.w;
                    } else {
                        c[0] = fmaf(wk, v.x, c[0]); c[1] = fmaf(wk, v.y, c[1]);
                        c[2] = fmaf(wk, v.z, c[2]); c[3] = fmaf(wk, v.w, c[3]);
                    }
                }
                color = make_float4(c[0], c[1], c[2], c[3]);
            }
        }
    } else {
        // ---- a3/a4 (COLLAB) or the pure STF / WC modes: decide who produces what
        Box b;
        b.fits = false;
        b.K = 0;
        b.lgP = 0;
        b.minx = b.miny = 0;
        int rho[4] = {0, 0, 0, 0}, n = 0xFF, fb;
        int box_w = 0, box_n = 0;   // Box variant: AABB width and area
        bool exact = false;
        if constexpr (MODE == MODE_COLLAB) {
            // collect the exact unique set U and canonical ranks
            b = wave_box(f, true);   // inactive lanes carry a duplicate footprint
            if (b.K == 1) n = collect_mask<1>(f, b, true, rho, s, lane);
            else if (b.K == 2) n = collect_mask<2>(f, b, true, rho, s, lane);
            else if (b.K == 4) n = collect_mask<4>(f, b, true, rho, s, lane);
            else {
                const Collected cc = collect_sort(f, true, s, lane, a.tex.W);
                n = cc.n;
#pragma unroll
                for (int k = 0; k < 4; ++k) rho[k] = cc.rho[k];
            }
            __syncwarp();
            // a4: List semantics exact iff n <= a (R-6).  The paper's Box and
            // Mask variants add AABB conditions.
            if (a.variant == VAR_LIST) {
                exact = n <= na;
            } else {
                const int bw = __reduce_max_sync(FULL, f.xb) - b.minx + 1;
                const int bh = __reduce_max_sync(FULL, f.yb) - b.miny + 1;
                if (a.variant == VAR_BOX) {
                    box_w = bw;
                    box_n = bw * bh;
                    exact = box_n <= na;
                } else {
                    const int lim = a.variant == VAR_MASK16 ? 16 : 11;
                    exact = bw <= lim && bh <= lim && n <= na;
                }
            }
            exact = exact && !(a.flags & FLAG_FORCE_FALLBACK);
            fb = a.fallback;
        } else {
            fb = MODE == MODE_STF ? FB_STF : FB_WC;
            if constexpr (MODE == MODE_WC) b = wave_box(f, active);
        }
        const bool full = A == FULL;
        Plan pl;
        if (exact) {
            // ---- a5: active rank r < n produces U[r] on lane h(r, A)
            const int ar = __popc(A & lt);
            if (!full) {
                if (active) s.lane_of_rank[ar] = (uint8_t)lane;
                __syncwarp();
            }
            pl.qx = pl.qy = 0;
            pl.selbits = 0u;
            if (a.variant != VAR_BOX) {
                pl.produced = active && ar < n;
                if (pl.produced) {
                    const uint32_t e = s.tbl[ar];
                    if (b.fits) { pl.qx = box_x(b, e); pl.qy = box_y(b, e); }
                    else { pl.qx = (int)(e & 0xffffu); pl.qy = (int)(e >> 16); }
                }
            } else {
                // Box: active rank i < w*h produces AABB texel (i mod w, i div w)
                // (LaneIdxToCoord); corners gather by their local index
                // (CoordToLaneIdx) through h(., A)
                pl.produced = active && ar < box_n;
                const int yq = ar / box_w;
                pl.qx = b.minx + (ar - yq * box_w);
                pl.qy = b.miny + yq;
                const int t0 = (f.ya - b.miny) * box_w + (f.xa - b.minx);
                const int t2 = (f.yb - b.miny) * box_w + (f.xa - b.minx);
                rho[0] = t0;
                rho[1] = t0 + (f.xb - f.xa);
                rho[2] = t2;
                rho[3] = t2 + (f.xb - f.xa);
            }
        } else if constexpr (FMT == FMT_BC1) {
            pl.produced = false;
            pl.qx = pl.qy = 0;
        } else {
            pl = fb_plan(fb, f, b, active, A, na, px, py + a.row0, frame, a.seed_lo, a.seed_hi, a.tex.W, s);
        }
        FbAll fball{};
        if constexpr (FMT == FMT_BC1) {
            if (!exact) fball = fb_all_bc1(fb, f, b, active, A, na, px, py + a.row0, frame, a, s);
        }
        selbits = (FMT == FMT_BC1 && !exact) ? fball.selbits : pl.selbits;
        // ---- the single texel-production site (<= 1 evaluation per lane)
        Texel<FMT> val = Texel<FMT>::zero();
        if constexpr (kBatchMlp) {
#if CTF_MLP_TC
            // exact and fallback waves alike: the wave's produced texels (row = lane)
            // go through the tensor-core decoder together
            val.v = mlp_decode_tc(a.tex, *mc.tw, *mc.tsc, pl.produced, pl.qx, pl.qy, lane);
            if (pl.produced) prod = (uint32_t)(pl.qy * a.tex.W + pl.qx);
#else
            if (exact) {
                MlpBatchSmem &ms = reinterpret_cast<MlpBatchSmem *>(mc.dyn)[mc.warp];
                val.v = mlp_decode_batched(a.tex, mw, ms, *mc.lw, pl.produced, __popc(A & lt), pl.qx, pl.qy,
                                           a.variant == VAR_BOX ? box_n : n, lane);
                if (pl.produced) prod = (uint32_t)(pl.qy * a.tex.W + pl.qx);
            } else if (pl.produced) {
                val = produce(a.tex, mw, pl.qx, pl.qy);
                prod = (uint32_t)(pl.qy * a.tex.W + pl.qx);
            }
#endif
        } else if (pl.produced) {
            val = produce(a.tex, mw, pl.qx, pl.qy);
            prod = (uint32_t)(pl.qy * a.tex.W + pl.qx);
        }
        if constexpr (FMT == FMT_BC1) {
            if (!exact) prod = fball.prod;
        }
        if (exact) {
            // evals = n (Box: the AABB area), path 0
            rec = rec_base | ((uint32_t)n << 8) | (uint32_t)(a.variant == VAR_BOX ? box_n : n);
            // ---- a6: gather from lanes h(rho_k, A) and blend
            int src[4];
            if (full) {
#pragma unroll
                for (int k = 0; k < 4; ++k) src[k] = rho[k];
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) src[k] = active ? (int)s.lane_of_rank[rho[k] & 31] : (int)lane;
            }
            Texel<FMT> p[4];
#if CTF_MLP_TC
            if constexpr (kBatchMlp) {
                // the tensor-core decoder left every lane's texel in its scratch row: one
                // LDS.128 per corner instead of four 32-bit shuffles
#pragma unroll
                for (int k = 0; k < 4; ++k) p[k].v = mc.tsc->out[src[k]];
            } else
#endif
            {
#pragma unroll
                for (int k = 0; k < 4; ++k) p[k] = Texel<FMT>::shfl(val, src[k]);
            }
            if (active) color = blend4<FMT>(p, f.w);
            if (DBG && a.dbg_unread) {
                unsigned bad = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int pk = __shfl_sync(FULL, (int)pl.produced, src[k]);  // every lane shuffles
                    bad += (active && !pk) ? 1u : 0u;
                }
                bad = __reduce_add_sync(FULL, bad);       // warp-uniform: no divergent atomic
                if (lane == 0 && bad) atomicAdd(a.dbg_unread, bad);
            }
        } else {
            // ---- a7: fallback combine
            Finished o;
            if constexpr (FMT == FMT_BC1) o = fball.fin;
            else o = fb_finish<FMT>(fb, f, b, active, na, pl, val, a.tex.W, s);
            color = o.color;
            const uint32_t path = MODE == MODE_COLLAB ? (uint32_t)(PATH_FB_STF + fb)
                                                      : (uint32_t)(MODE == MODE_STF ? PATH_STF : PATH_WC);
            rec = rec_base | ((uint32_t)(n & 0xFF) << 8) | (path << 22) | (uint32_t)(o.evals & 0xFF);
        }
    }

    return {color, rec, prod, selbits};
}

template <int FMT, int MODE, bool DBG>
__global__ void __launch_bounds__(kWarps * 32, (FMT == FMT_BC1 ? CTF_BC1_MINB : (MODE == MODE_COLLAB ? CTF_MLP_COLLAB_MINB : 2)))
    ctf_filter_kernel(const KArgs a, const typename WeightsOf<FMT>::type mw) {
    __shared__ WarpSmem smem[kWarps];
    extern __shared__ __align__(16) unsigned char dyn_smem[];   // latent-MLP COLLAB: batch buffers
    const unsigned lane = lane_id(), warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);   // provably warp-uniform (no divergence guards)
    WarpSmem &s = smem[warp];
    constexpr bool kBatchMlp = FMT == FMT_MLP && MODE == MODE_COLLAB;
    MlpCtx mc{nullptr, nullptr, nullptr, dyn_smem, warp};
#if CTF_MLP_TC
    // tensor-core decoder: weights (hi / lo fp16) shared by the CTA, scratch per warp
    TcWeights &tw = *reinterpret_cast<TcWeights *>(dyn_smem);
    TcScratch &tsc = reinterpret_cast<TcScratch *>(dyn_smem + sizeof(TcWeights))[warp];
    if constexpr (kBatchMlp) fill_tc_weights(mw, tw);
    mc.tw = &tw;
    mc.tsc = &tsc;
#else
    MlpLaneWeights lw;
    if constexpr (kBatchMlp) load_lane_weights(a.tex.mlp_dev, lane, lw);
    mc.lw = &lw;
#endif
    const int lx = (int)(lane & 7), ly = (int)(lane >> 3);

    // work item c = (frame, wave-row, run of kChunk waves); items are interleaved over
    // the whole batch so every warp gets the same mix of sky / exact / fallback regions.
    //   BC1: warp (b, w) takes items b*kWarps + w + j*gridDim.x*kWarps, j < ipc/kWarps
    //        (short static lists; the grid is many CTAs and the block scheduler balances);
    //   MLP: one CTA per slot, CTA b owns items b + k*gridDim.x and its warps claim k
    //        from a shared counter (long items, per-warp weight preload).
    __shared__ unsigned s_next;
    if constexpr (FMT != FMT_BC1) {
        if (threadIdx.x == 0) s_next = kWarps;
        __syncthreads();
    }
    const unsigned per_warp = a.ipc / kWarps;
    for (unsigned k = warp;;) {
        const unsigned c = (FMT == FMT_BC1)
                               ? (blockIdx.x * kWarps + (k % kWarps)) + (k / kWarps) * gridDim.x * kWarps
                               : blockIdx.x + k * gridDim.x;
        if ((FMT == FMT_BC1 ? k / kWarps >= per_warp : k >= a.ipc) || c >= a.nchunks) break;
        if constexpr (FMT == FMT_BC1) {
            k += kWarps;
        } else {
            unsigned nx = 0u;
            if (lane == 0) nx = atomicAdd(&s_next, 1u);
            k = __shfl_sync(FULL, nx, 0);
        }
        const int fr = (int)(c / (unsigned)a.cpf);
        const int rr = (int)(c - (unsigned)fr * (unsigned)a.cpf);
        const int wy = rr / a.cpr;
        const int wx0 = (rr - wy * a.cpr) * a.chunk;
        const int wx1 = min(wx0 + a.chunk, a.nwx);
        const int py = wy * 4 + ly;
        const bool rowok = py < a.Hf;
        const uint32_t frame = a.frame_index + (uint32_t)fr;
        unsigned w = (unsigned)fr * (unsigned)a.wpf + (unsigned)(wy * a.nwx + wx0);    // record index
        unsigned pix = (unsigned)fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)(wx0 * 8 + lx);
        int px = wx0 * 8 + lx;

        // software pipeline: wave wx+1's uv/grad loads are issued before wave wx is
        // processed, so their HBM latency hides behind this wave's work
        const bool has_grad = a.grad != nullptr;
        float2 uv_n = make_float2(__int_as_float(0x7fc00000), 0.f);
        uint2 gr_n = make_uint2(0u, 0u);
        ld_stream_f2_if(uv_n, a.uv + pix, rowok & (px < a.Wf));
        ld_stream_u2_if(gr_n, a.grad + pix, rowok & (px < a.Wf) & has_grad);
        uint32_t myrec = 0u;  // record of wave wx0 + lane, stored once per run
        const unsigned w0 = w;
        for (int wx = wx0; wx < wx1; ++wx, ++w, pix += 8u, px += 8) {
            const bool inframe = rowok & (px < a.Wf);
            const float2 uv = uv_n;
            const uint2 gr = gr_n;
            // (no reset needed: lanes whose next pixel is outside the frame are inactive there)
            const bool pf = (wx + 1 < wx1) & rowok & (px + 8 < a.Wf);
            ld_stream_f2_if(uv_n, a.uv + (pix + 8u), pf);
            ld_stream_u2_if(gr_n, a.grad + (pix + 8u), pf & has_grad);

            __syncwarp();  // order this wave's shared-memory tables after the previous wave's reads
            // ---- a1: classify
            const bool active = inframe && !isnan(uv.x);
            const unsigned A = __ballot_sync(FULL, active);
            const int na = __popc(A);
            if (na == 0) {
                if (inframe) st_stream_f4(a.out + pix, make_float4(0.f, 0.f, 0.f, 0.f));
                if (DBG && inframe) {
                    if (a.dbg_pid) a.dbg_pid[pix] = INVALID_ID;
                    if (a.dbg_sel) a.dbg_sel[pix] = 0u;
                }
                if (lane == (unsigned)(wx - wx0)) myrec = ((MODE == MODE_COLLAB ? 0u : 0xFFu) << 8) | (1u << 26);
                continue;
            }
            const WaveOut o = wave_general<FMT, MODE, DBG>(a, mw, s, mc, uv, gr, active, A, na, px, py, frame);
            // ---- outputs
            if (inframe) st_stream_f4(a.out + pix, o.color);
            if (DBG && inframe) {
                if (a.dbg_pid) a.dbg_pid[pix] = (MODE == MODE_4TAP) ? INVALID_ID : o.prod;
                if (a.dbg_sel) a.dbg_sel[pix] = o.selbits;
            }
            // ---- a8: per-wave record (kept in lane wx - wx0, stored per run)
            if (lane == (unsigned)(wx - wx0)) myrec = o.rec;
        }
        if (lane < (unsigned)(wx1 - wx0)) a.rec[w0 + lane] = myrec;
    }
}

// ---------------------------------------------- COLLAB (List) kernels: the lean path
// On a magnified frame nearly every wave is FULL (32 active lanes) with a footprint
// bounding box that fits an 8x4 / 4x8 window (one 32-bit mask) or an 8x8 window (two
// words).  Those waves run the straight-line code below, exact or fallback:
//   collect  : 2 redux.min (AABB origin) + 1-3 votes (window) + 1-2
//              redux.or (WaveActiveBitOr) + popc ranks (h^-1);
//   decide   : exact iff n <= 32 (the wave is full);
//   produce  : exact: lane r < n decodes U[r] (h(r, A) = r); fallback: the
//              STF / C+ plan below; one decode site, converted to fp32 once (v / 255);
//   gather   : the produced values go through shared memory (one STS.128 per producer,
//              LDS.128 per corner) — WaveReadLaneAt with the conversion
//              done once per texel instead of once per read;
//   filter   : exact: blend4f (FFMA2), bit-identical to every other exact path;
//              fallback: one-tap / WC / Eq. 1 (combine_eq1f, as the general path).
// The waves the lean kernel does not finish are marked in their record and finished by
// two more kernels that use the record buffer as their work list (no workspace):
//   kFbMark   full waves whose window fits 8x8 but need a fallback (n > 32) ->
//             the same lean code with the fallback enabled (64 registers, no spills);
//   kSlowMark partial waves and wider windows (minified waves) -> the general path
//             (wave_general, 80 registers).
// The lean kernel itself contains no call and no fallback code (a call or a divergent
// region before a warp collective makes ptxas guard every collective of the loop with a
// divergence check).
constexpr uint32_t kSlowMark = 0xFFFFFFFFu;   // neither is a COLLAB record (path <= 4, n <= 128)
constexpr uint32_t kFbMark = 0xFFFFFFFEu;
#ifndef CTF_REST_ROWS
#define CTF_REST_ROWS 32  // window rows of the wide-window kernel's bitmap (32 or 64)
#endif
#ifndef CTF_REST_CONCURRENT
#define CTF_REST_CONCURRENT 1  // BC1: the lean kernel routes each wave it leaves by its AABB (the wide-window
                               // kernel's 32 x CTF_REST_ROWS window, else the third kernel), so the third kernel
                               // runs first and the wide-window kernel alongside it (PDL, see launch_rest)
#endif
// BC1, a wave the lean path leaves: kFbMark when its active lanes' footprint AABB fits the
// wide-window kernel's window, else kSlowMark (the third kernel's 64 x 64 window / general path)
// — the same test as wide_wave's, so the wide-window kernel never re-marks a wave
__device__ __forceinline__ uint32_t bc1_rest_mark(const Foot &f, bool active) {
    if (!CTF_REST_CONCURRENT) return kFbMark;
    const int minx = __reduce_min_sync(FULL, active ? f.xa : INT_MAX);
    const int miny = __reduce_min_sync(FULL, active ? f.ya : INT_MAX);
    const int maxx = __reduce_max_sync(FULL, active ? f.xb : INT_MIN);
    const int maxy = __reduce_max_sync(FULL, active ? f.yb : INT_MIN);
    return (maxx - minx >= 32 || maxy - miny >= CTF_REST_ROWS) ? kSlowMark : kFbMark;
}

struct FastSmem {
    float4 xch[32];           // rank -> produced value (exact waves, n <= 32)
    uint4 lut[8];             // BC1 per-index constants (bc1_lut_entry), per warp
    uint8_t bit_of_rank[32];  // rank -> window bit (0..63)
};

#ifndef CTF_FAST_MINB
#define CTF_FAST_MINB 7  // resident CTAs per SM (32 registers, no spills)
#endif
#ifndef CTF_PAIR
#define CTF_PAIR 1  // BC1 non-debug: two waves share one decode pass (pair_front / pair_decode)
#endif
#ifndef CTF_PAIR_MLP
#define CTF_PAIR_MLP 1  // latent MLP non-debug: two waves share one tensor-core decode
#endif
#ifndef CTF_PAIR_MINB
#define CTF_PAIR_MINB 6  // paired lean kernel: resident CTAs per SM (40 registers)
#endif


// Shared memory of the paired exact path: wave A's produced texels take jobs 0..nA-1,
// wave B's jobs nA..nA+nB-1 (xch / bit_of_rank indexed by job).
struct PairSmem {
    float4 xch[64];           // job -> produced value
    uint4 lut[8];             // BC1 per-index constants (bc1_lut_entry), per warp
    uint8_t bit_of_rank[96];  // job -> window offset (dy << 3) | dx; [64, 96): per-lane scratch slots
};

// 64-bit window masks held as two words (hi = 0 for a 32-bit window)
__device__ __forceinline__ uint32_t bit_lo(uint32_t t) { return t < 32u ? 1u << t : 0u; }
__device__ __forceinline__ uint32_t bit_hi(uint32_t t) { return t >= 32u ? 1u << (t - 32u) : 0u; }
__device__ __forceinline__ int rank64(uint32_t lo, uint32_t hi, uint32_t t) {   // set bits below t
    return t < 32u ? __popc(lo & ((1u << t) - 1u)) : __popc(lo) + __popc(hi & ((1u << (t - 32u)) - 1u));
}

// Distinct texels of a footprint and their merged fp32 weights (R-14) from the clamp
// flags alone: corner k is the first occurrence of its texel iff (k & 1 -> xb != xa) and
// (k & 2 -> yb != ya), and the duplicates are added in corner order — the same values,
// bit for bit, as distinct_corners() (adding +0 is exact).
struct Merged {
    float dw[4];
    bool first[4];
};
__device__ __forceinline__ Merged merge_corners(const Foot &f) {
    const bool ddx = f.xb != f.xa, ddy = f.yb != f.ya;
    Merged m;
    m.dw[0] = __fadd_rn(__fadd_rn(__fadd_rn(f.w[0], ddx ? 0.0f : f.w[1]), ddy ? 0.0f : f.w[2]),
                        (ddx || ddy) ? 0.0f : f.w[3]);
    m.dw[1] = __fadd_rn(f.w[1], ddy ? 0.0f : f.w[3]);
    m.dw[2] = __fadd_rn(f.w[2], ddx ? 0.0f : f.w[3]);
    m.dw[3] = f.w[3];
    m.first[0] = true;
    m.first[1] = ddx;
    m.first[2] = ddy;
    m.first[3] = ddx && ddy;
    return m;
}

// bit k = corner k is the first occurrence of its texel and its merged weight is nonzero
__device__ __forceinline__ unsigned contrib_bits(const Foot &f, const Merged &m) {
    const unsigned ddx = f.xb != f.xa, ddy = f.yb != f.ya;
    const unsigned first = 1u | (ddx << 1) | (ddy << 2) | ((ddx & ddy) << 3);
    const unsigned nz = (m.dw[0] != 0.0f ? 1u : 0u) | (m.dw[1] != 0.0f ? 2u : 0u) | (m.dw[2] != 0.0f ? 4u : 0u) |
                        (m.dw[3] != 0.0f ? 8u : 0u);
    return first & nz;
}

// One-tap-free Eq. 1 / WC stand-in from the four corner values pv[k] (0 where the texel
// was not produced; IN = produced corner mask).  Same operations in the same order as
// combine_eq1f over distinct_corners — fma by an exact 0 / 1 adds nothing / exactly p —
// so the special cases (all known -> exact bilinear; N = 1 -> that texel) hold bit for
// bit and the rest equals it.
template <bool WC>
__device__ __forceinline__ float4 combine_eq1_mc(const Foot &f, const Merged &m, unsigned C, unsigned IN,
                                                 const float4 (&pv)[4]) {
    const unsigned Kn = C & IN;
    const bool all_known = (C & ~IN) == 0u;
    const int N = __popc(Kn);
    float Sw = 0.0f;
    uint64_t sp01 = f2pack(0.f, 0.f), sp23 = f2pack(0.f, 0.f), sq01 = f2pack(0.f, 0.f), sq23 = f2pack(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool kn = (Kn >> k) & 1u;
        const float one = kn ? 1.0f : 0.0f, wk = kn ? m.dw[k] : 0.0f;
        Sw = __fadd_rn(Sw, wk);
        sp01 = ffma2(f2pack(pv[k].x, pv[k].y), f2pack(one, one), sp01);   // Sp += p (exact product)
        sp23 = ffma2(f2pack(pv[k].z, pv[k].w), f2pack(one, one), sp23);
        if (WC) {
            sq01 = ffma2(f2pack(pv[k].x, pv[k].y), f2pack(wk, wk), sq01);   // sum dw * p
            sq23 = ffma2(f2pack(pv[k].z, pv[k].w), f2pack(wk, wk), sq23);
        }
    }
    const float4 bl = blend4f(pv, f.w);   // sum over the known corners of w_k p_k
    const float2 a01 = f2unpack(sp01), a23 = f2unpack(sp23);
    float4 c;
    if (WC) {
        const float2 q01 = f2unpack(sq01), q23 = f2unpack(sq23);
        const float r = 1.0f / Sw;
        c = all_known ? bl : make_float4(q01.x * r, q01.y * r, q23.x * r, q23.y * r);
    } else {
        const float rest = (all_known || N == 0) ? 0.0f : __fdividef(1.0f - Sw, (float)N);
        c = make_float4(fmaf(rest, a01.x, bl.x), fmaf(rest, a01.y, bl.y), fmaf(rest, a23.x, bl.z),
                        fmaf(rest, a23.y, bl.w));
    }
    if (N == 1 && !all_known) c = make_float4(a01.x, a01.y, a23.x, a23.y);
    return c;
}
// Eq. 1 as one 4-corner blend with per-corner coefficients: a known corner k
// contributes w_k (its duplicates too: their sum is the merged weight of the texel, R-14) plus,
// on the first occurrence of each known nonzero-weight texel, rest = (1 - Sum_K dw) / N, so the
// blend is Sum_K dw p + rest * Sum_K p; unknown corners get 0.  The special cases hold up to
// fp32 rounding: all known -> rest = 0 and the blend is the exact-path chain; N = 1 ->
// (dw + (1 - dw)) p.  pv must be finite everywhere (coefficient 0 x value).
__device__ __forceinline__ float4 combine_eq1_coef(const Foot &f, const Merged &m, unsigned C, unsigned IN,
                                                   const float4 (&pv)[4]) {
    const unsigned Kn = C & IN;
    const bool all_known = (C & ~IN) == 0u;
    const int N = __popc(Kn);
    float Sw = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) Sw = __fadd_rn(Sw, ((Kn >> k) & 1u) ? m.dw[k] : 0.0f);
    const float rest = (all_known || N == 0) ? 0.0f : __fdividef(1.0f - Sw, (float)N);
    float cf[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        cf[k] = __fadd_rn(((IN >> k) & 1u) ? f.w[k] : 0.0f, ((Kn >> k) & 1u) ? rest : 0.0f);
    return blend4f(pv, cf);
}

// One FULL wave (32 active lanes) through the lean exact path.  Returns done = false with
// rec = kFbMark when the wave needs a fallback or its window only fits a 128-bit shape
// (16x8, 8x16, 32x4), or kSlowMark when no window fits (general path).
struct LeanOut {
    float4 color;
    uint32_t rec, prod, selbits;
    bool done;   // else rec = the mark for the kernel that finishes the wave
};

// magnified class of a full wave (R-20), as in the general path
__device__ __forceinline__ bool wave_magnified(uint2 gr, bool has_grad) {
    bool mag_lane = true;
    if (has_grad) {
        const float rx = fma_f32_f16((unsigned short)(gr.x & 0xffffu), (unsigned short)(gr.x & 0xffffu),
                                     fma_f32_f16((unsigned short)(gr.x >> 16), (unsigned short)(gr.x >> 16), 0.0f));
        const float ry = fma_f32_f16((unsigned short)(gr.y & 0xffffu), (unsigned short)(gr.y & 0xffffu),
                                     fma_f32_f16((unsigned short)(gr.y >> 16), (unsigned short)(gr.y >> 16), 0.0f));
        mag_lane = rx <= 1.0f && ry <= 1.0f;
    }
    return has_grad && __all_sync(FULL, mag_lane);
}

// FMT_MLP: the wave's produced texels go through the tensor-core decoder together
// (mlp_decode_tc, rows = lanes); its fallback and 128-bit-window waves go to the general
// kernel (kSlowMark) — there is no lean fallback for the latent-MLP format.
// BOX: Box Sampling: exact iff the AABB area w*h <= a = 32; job j < w*h decodes
// AABB texel (j mod w, j div w) (LaneIdxToCoord), a corner reads its AABB-local
// index (CoordToLaneIdx); n (unique texels) goes to the record only.  The lean
// windows are <= 8 wide and tall, so j div w = trunc((j + 1/2) / w) in fp32 is exact.
__device__ __forceinline__ int box_row(unsigned j, int w) { return (int)__fdividef((float)j + 0.5f, (float)w); }

template <bool DBG, int FMT, class SM, bool BOX = false>
__device__ __forceinline__ LeanOut lean_wave(const KArgs &a, SM &fs, const uint4 *lut, const MlpCtx &mc,
                                             float2 uv, uint2 gr, bool has_grad) {
    const unsigned lane = lane_id(), lt = lanemask_lt(), lanebit = 1u << lane;
    LeanOut o;
    o.color = make_float4(0.f, 0.f, 0.f, 0.f);
    o.rec = kFbMark;
    o.prod = INVALID_ID;
    o.selbits = 0u;
    o.done = false;
    // ---- a1: magnified class
    const bool wave_mag = wave_magnified(gr, has_grad);
    // ---- a2: footprint (packed fp32; = footprint())
    const Foot f = footprint2(uv, a);
    // ---- a3: AABB origin and window
    const int minx = __reduce_min_sync(FULL, f.xa), miny = __reduce_min_sync(FULL, f.ya);
    const unsigned dx = (unsigned)(f.xb - minx), dy = (unsigned)(f.yb - miny);
    int K = 0;
    unsigned lgP = 3u;
    if (__all_sync(FULL, (dx | (dy << 1)) < 8u)) K = 1;                      // 8x4
    else if (__all_sync(FULL, (dy | (dx << 1)) < 8u)) { K = 1; lgP = 2u; }   // 4x8
    else if (__all_sync(FULL, (dx | dy) < 8u)) K = 2;                        // 8x8
    if (K == 0) {   // a wider window: the wide-window kernel / the third kernel (BC1), the general kernel (latent MLP)
        o.rec = FMT == FMT_BC1 ? bc1_rest_mark(f, true) : kSlowMark;
        return o;
    }
    const uint32_t pmask = (1u << lgP) - 1u;
    const uint32_t t0 = ((uint32_t)(f.ya - miny) << lgP) + (uint32_t)(f.xa - minx);
    const uint32_t t2 = t0 + ((uint32_t)(f.yb - f.ya) << lgP);
    const uint32_t dxs = (uint32_t)(f.xb - f.xa);
    const uint32_t pat = 1u + dxs + dxs;   // bits t and t + dxs (same window row)
    int n, r0, r2;
    if (K == 1) {
        const uint32_t wm = __reduce_or_sync(FULL, (pat << t0) | (pat << t2));
        n = __popc(wm);
        r0 = __popc(wm & ((1u << t0) - 1u));
        r2 = __popc(wm & ((1u << t2) - 1u));
        if (!BOX) st_shared_u8_if(fs.bit_of_rank + __popc(wm & lt), lane, wm & lanebit);
    } else {
        const uint64_t m = ((uint64_t)pat << t0) | ((uint64_t)pat << t2);
        const uint32_t wl = __reduce_or_sync(FULL, (uint32_t)m);
        const uint32_t wh = __reduce_or_sync(FULL, (uint32_t)(m >> 32));
        const int nl = __popc(wl);
        n = nl + __popc(wh);
        r0 = rank64(wl, wh, t0);
        r2 = rank64(wl, wh, t2);
        if (!BOX) {
            st_shared_u8_if(fs.bit_of_rank + __popc(wl & lt), lane, wl & lanebit);
            const int rh = nl + __popc(wh & lt);
            st_shared_u8_if(fs.bit_of_rank + (rh & 31), 32u + lane, (wh & lanebit) && rh < 32);
        }
    }
    int evals = n;   // jobs: n (List), the AABB area (Box)
    if constexpr (BOX) {
        const int bw = (int)__reduce_max_sync(FULL, dx) + 1, bh = (int)__reduce_max_sync(FULL, dy) + 1;
        evals = bw * bh;
        if (evals > 32) {   // Box fallback: lean fallback kernel (BC1) / general kernel (latent MLP)
            if (FMT != FMT_BC1) o.rec = kSlowMark;
            return o;
        }
        const int jq = box_row(lane, bw);
        st_shared_u8_if(fs.bit_of_rank + lane, ((uint32_t)jq << lgP) | (lane - (uint32_t)(jq * bw)), (int)lane < evals);
        r0 = (f.ya - miny) * bw + (f.xa - minx);
        r2 = r0 + (f.yb - f.ya) * bw;
    } else if (n > 32) {   // ---- a4: exact iff n <= a = 32 (always for a 32-bit window)
        if (FMT != FMT_BC1) o.rec = kSlowMark;   // fallback kernel (BC1) / general kernel (latent MLP)
        return o;
    }
    o.done = true;
    __syncwarp();
    // ---- a5: lane r < n produces U[r] (h(r, A) = r); one decode site, fp32 once
    // (SIMT: the decoder runs on every lane; non-producers decode the window origin and
    // do not store — predicated, so the loop stays free of divergent regions)
    const bool produced = (int)lane < evals;
    const uint32_t e = produced ? (uint32_t)fs.bit_of_rank[lane] : 0u;
    const int qx = minx + (int)(e & pmask), qy = miny + (int)(e >> lgP);
    const float4 *xv;   // rank -> produced value
    if constexpr (FMT == FMT_BC1) {
        st_shared_f4_if(&fs.xch[lane], bc1_decode_unorm_lut(a.tex, qx, qy, lut), produced);
        xv = fs.xch;
    } else {
        // rows = lanes = ranks; the decoder leaves every row's texel in its scratch
        mlp_decode_tc(a.tex, *mc.tw, *mc.tsc, produced, qx, qy, lane_id());
        xv = mc.tsc->out;
    }
    if (DBG) o.prod = produced ? (uint32_t)(qy * a.tex.W + qx) : INVALID_ID;
    __syncwarp();
    // ---- a6: gather (ranks rho_k) + blend
    const float4 p[4] = {xv[r0], xv[r0 + (int)dxs], xv[r2], xv[r2 + (int)dxs]};
    o.color = blend4f(p, f.w);
    o.rec = ((uint32_t)n << 8) | (uint32_t)evals | (32u << 16) | ((uint32_t)wave_mag << 25);
    if (DBG && a.dbg_unread) {
        const unsigned bad = __reduce_add_sync(FULL, (unsigned)(r0 >= evals) + (unsigned)(r0 + (int)dxs >= evals) +
                                                         (unsigned)(r2 >= evals) + (unsigned)(r2 + (int)dxs >= evals));
        if (lane == 0 && bad) atomicAdd(a.dbg_unread, bad);
    }
    return o;
}

// ------------------------------------------- paired exact path (non-debug build)
// Two consecutive waves of a run share one decode pass.  Each wave still evaluates exactly
// its own unique set U (n texels; its rank r is job base + r, h(r, A) = r up to the
// offset), so colours, records and evaluation counts equal the one-wave path bit
// for bit; only the SIMT packing of the evaluations changes: with n ~ 13 per wave (config
// 5) one 32-lane decode pass serves both waves (two passes when nA + nB > 32).
struct PairFront {
    float s, t;        // footprint fractions (the weights are rebuilt from them, as footprint2)
    uint32_t a0, a2;   // shared addresses of xch[job of the upper-left / lower-left corner]
    uint32_t dxs16;    // 16 * (xb - xa): the right corners' slots follow the left ones
    int n;             // produced texels; 0: the wave is not finished here (rec says where)
    int minx, miny;    // window origin
    uint32_t rec;
};
// steps a1-a4 of lean_wave for one wave; the rank -> window-bit table goes to job base + r
// the push-table codes (dy << 3) | dx of window bit `lane` for the pitches P = 8, 4, 6, 5, one
// byte each (computed once per thread; pair_front selects a byte by the window's pitch)
__device__ __forceinline__ uint32_t push_codes(unsigned lane) {
    uint32_t c = 0u;
    const unsigned P[4] = {8u, 4u, 6u, 5u};
#pragma unroll
    for (int i = 0; i < 4; ++i) c |= (((lane / P[i]) << 3) | (lane % P[i])) << (8 * i);
    return c;
}
template <bool GRAD, int FMT, class SM, bool BOX = false>
__device__ __forceinline__ PairFront pair_front(const KArgs &a, SM &fs, float2 uv, uint2 gr, int base, uint8_t *bits0,
                                                unsigned lane, unsigned lt, uint32_t cpk) {
    const unsigned lanebit = 1u << lane;
    PairFront o;
    o.s = o.t = 0.f;
    o.a0 = o.a2 = o.dxs16 = 0u;
    o.n = 0;
    o.minx = o.miny = 0;
    const unsigned A = __ballot_sync(FULL, !isnan(uv.x));   // interior run: every pixel in the frame
    if (A != FULL) {   // empty wave: n = 0, zero colour; partial wave: wide-window / third kernel (BC1)
        o.rec = A == 0u ? (1u << 26) : (FMT == FMT_BC1 ? bc1_rest_mark(footprint2(uv, a), !isnan(uv.x)) : kSlowMark);
        return o;
    }
    const bool wave_mag = wave_magnified(gr, GRAD);
    const Foot f = footprint2(uv, a);
    const int minx = __reduce_min_sync(FULL, f.xa), miny = __reduce_min_sync(FULL, f.ya);
    const unsigned dx = (unsigned)(f.xb - minx), dy = (unsigned)(f.yb - miny);
    // window P x (32 / P) or 8 x 8, row-major (bit t = dy * P + dx: the rank order is the
    // row-major order of U for every shape); 6x5 / 5x6 take the 5x5..6x6 AABBs of rotated
    // magnified waves (~10 % of config-5 waves) off the 64-bit path
    int K = 0;
    uint32_t P = 8u, csel = 0x4440u;   // pitch; byte_perm selector of cpk's byte holding this pitch's push code
    if (__all_sync(FULL, (dx | (dy << 1)) < 8u)) K = 1;                                    // 8x4
    else if (__all_sync(FULL, (dy | (dx << 1)) < 8u)) { K = 1; P = 4u; csel = 0x4441u; }   // 4x8
    else if (__all_sync(FULL, dx < 6u && dy < 5u)) { K = 1; P = 6u; csel = 0x4442u; }      // 6x5
    else if (__all_sync(FULL, dx < 5u && dy < 6u)) { K = 1; P = 5u; csel = 0x4443u; }      // 5x6
    else if (__all_sync(FULL, (dx | dy) < 8u)) K = 2;                                      // 8x8
    if (K == 0) {   // a wider window: the wide-window / third kernel (BC1), the general kernel (latent MLP)
        o.rec = FMT == FMT_BC1 ? bc1_rest_mark(f, true) : kSlowMark;
        return o;
    }
    const uint32_t t0 = (uint32_t)(f.ya - miny) * P + (uint32_t)(f.xa - minx);
    const uint32_t t2 = t0 + (uint32_t)(f.yb - f.ya) * P;
    const uint32_t dxs = (uint32_t)(f.xb - f.xa);
    const uint32_t pat = 1u + dxs + dxs;
    // push table entry of window bit t: its offset (dy << 3) | dx from the window origin
    const uint32_t code = __byte_perm(cpk, 0u, csel);   // = ((lane / P) << 3) | (lane % P)
    uint8_t *bits = bits0 + base;
    int n, r0, r2;
    if (K == 1) {
        const uint32_t wm = __reduce_or_sync(FULL, (pat << t0) | (pat << t2));
        n = __popc(wm);
        // rank of window bit t = set bits below t = lane t's popc(wm & lanemask_lt): the
        // corners' ranks are two shuffles of the push rank
        const int myr = __popc(wm & lt);
        r0 = __shfl_sync(FULL, myr, (int)t0);
        r2 = __shfl_sync(FULL, myr, (int)t2);
        // push (no predicate): the owner of window bit `lane` writes its code at its rank, every
        // other lane into its own scratch slot 64 + lane (no divergent store region)
        if (!BOX) bits0[(wm & lanebit) ? base + myr : 64 + (int)lane] = (uint8_t)code;
    } else {
        const uint64_t m = ((uint64_t)pat << t0) | ((uint64_t)pat << t2);
        const uint32_t wl = __reduce_or_sync(FULL, (uint32_t)m);
        const uint32_t wh = __reduce_or_sync(FULL, (uint32_t)(m >> 32));
        const int nl = __popc(wl);
        n = nl + __popc(wh);
        r0 = rank64(wl, wh, t0);
        r2 = rank64(wl, wh, t2);
        if (!BOX) {
            bits0[(wl & lanebit) ? base + __popc(wl & lt) : 64 + (int)lane] = (uint8_t)lane;
            const int rh = nl + __popc(wh & lt);
            bits0[((wh & lanebit) && rh < 32) ? base + (rh & 31) : 64 + (int)lane] = (uint8_t)(32u + lane);
        }
    }
    int evals = n;   // jobs: n (List), the AABB area (Box, see lean_wave)
    if constexpr (BOX) {
        const int bw = (int)__reduce_max_sync(FULL, dx) + 1, bh = (int)__reduce_max_sync(FULL, dy) + 1;
        evals = bw * bh;
        if (evals > 32) {   // Box fallback: lean fallback kernel (BC1) / general kernel (latent MLP)
            o.rec = FMT == FMT_BC1 ? kFbMark : kSlowMark;
            return o;
        }
        const int jq = box_row(lane, bw);
        st_shared_u8_if(bits + lane, ((uint32_t)jq << 3) | (lane - (uint32_t)(jq * bw)), (int)lane < evals);
        r0 = (f.ya - miny) * bw + (f.xa - minx);
        r2 = r0 + (f.yb - f.ya) * bw;
    } else if (n > 32) {   // fallback kernel (BC1) / general kernel (latent MLP)
        o.rec = FMT == FMT_BC1 ? kFbMark : kSlowMark;
        return o;
    }
    o.s = f.s;
    o.t = f.t;
    const uint32_t x0 = (uint32_t)__cvta_generic_to_shared(fs.xch + base);
    o.a0 = x0 + 16u * (uint32_t)r0;
    o.a2 = x0 + 16u * (uint32_t)r2;
    o.dxs16 = 16u * dxs;
    o.n = evals;
    o.minx = minx;
    o.miny = miny;
    // (n << 8) | evals | (32 << 16) | (mag << 25); List: evals = n, so n * 257 + constant
    o.rec = BOX ? (((uint32_t)n << 8) | (uint32_t)evals | (32u << 16) | ((uint32_t)wave_mag << 25))
                : (uint32_t)n * 257u + (wave_mag ? (32u << 16) | (1u << 25) : (32u << 16));
    return o;
}
// step a5 for both waves: job j < nA decodes wave A's U[j], job nA + r wave B's U[r]
// (latent MLP: the jobs of a pass are the rows of one tensor-core decode, mlp_decode_tc,
// which runs one 16-row M tile when the pass has <= 16 jobs)
template <int FMT, class SM>
__device__ __forceinline__ void pair_decode(const KArgs &a, SM &fs, const uint8_t *bits, const PairFront &A,
                                            const PairFront &B, unsigned lane, const MlpCtx &mc) {
    const int J = A.n + B.n;
    for (int j0 = 0; j0 < J; j0 += 32) {   // one pass, two when nA + nB > 32 (warp-uniform)
        const int j = j0 + (int)lane;
        const bool produced = j < J, inA = j < A.n;
        const uint32_t e = produced ? (uint32_t)bits[j] : 0u;   // (dy << 3) | dx
        const int qx = (inA ? A.minx : B.minx) + (int)(e & 7u);
        const int qy = (inA ? A.miny : B.miny) + (int)(e >> 3);
        if constexpr (FMT == FMT_BC1) {
            st_shared_f4_if(&fs.xch[j], bc1_decode_unorm_lut(a.tex, qx, qy, fs.lut), produced);
        } else {
            const float4 v = mlp_decode_tc(a.tex, *mc.tw, *mc.tsc, produced, qx, qy, lane);
            st_shared_f4_if(&fs.xch[j], v, produced);
        }
    }
}
// step a6 for one wave: gather + blend (weights as footprint2) and store; the empty wave
// stores its zero colour
template <class SM>
__device__ __forceinline__ void pair_back(const KArgs &a, const SM &fs, const PairFront &w, unsigned pix) {
    if (w.n > 0) {
        const float2 om = f2unpack(fsub2(f2pack(1.0f, 1.0f), f2pack(w.s, w.t)));
        const float wt[4] = {__fmul_rn(om.x, om.y), __fmul_rn(w.s, om.y), __fmul_rn(om.x, w.t), __fmul_rn(w.s, w.t)};
        const float4 p[4] = {ld_shared_f4(w.a0), ld_shared_f4(w.a0 + w.dxs16), ld_shared_f4(w.a2),
                             ld_shared_f4(w.a2 + w.dxs16)};
        st_stream_f4(a.out + pix, blend4f(p, wt));
    } else if (w.rec == (1u << 26)) {
        st_stream_f4(a.out + pix, make_float4(0.f, 0.f, 0.f, 0.f));
    }
}

// ------------------------------------------------ wide-window path (shared-memory bitmaps)
// Every wave the lean exact kernel leaves (n > 32, windows wider than 8x8, partial waves,
// forced fallbacks) whose footprint AABB fits 32 x ROWS texels: the window is a bitmap of ROWS
// rows x 32 bits in shared memory, one word per row, and each active lane sets its corners
// with two shared atomics (ATOMS.OR, one per footprint row) — the cost does not grow with
// the AABB (no 128-key sort).  The canonical ascending-id order (R-5) is row-major over the
// window, so a texel's rank is an exclusive scan of the rows' popcounts plus a popc within
// its row; a texel's rank and position do not depend on the lane that holds it, so every
// lane publishes its own texels (lanes sharing one store the same value; the atomics need no
// return value).  Bitmaps: U (the needed set: n and the exact ranks), P (the C+ plan), D (the
// produced set the fallbacks gather from: each producing lane stores its value in its own
// slot, the first producer of a texel — the D atomic's old value — its lane in a position ->
// lane table).  Records, producers, selections and colours equal the general path
// bit for bit (same fp32 operations in the same order).
// ROWS = 32 (lane l holds row l in the row scans; taller AABBs take the general path) or 64
// (lane l holds rows 2l and 2l + 1; CTF_REST_ROWS=64 builds the wide-window kernel that way).
// The general path evaluates Eq. 1 with the same coefficient blend (combine_eq1f), so the
// result does not depend on which path a wave takes.
template <int ROWS, int COLS = 32>
struct WideSmemT {
    static constexpr int kRows = ROWS, kCols = COLS, kCW = COLS / 32;   // kCW words per window row
    static_assert((ROWS == 32 || ROWS == 64) && (COLS == 32 || COLS == 64), "window shape");
    // window rows, row-major: bit (c & 31) of word r * kCW + (c >> 5) = texel (minx + c, miny + r)
    uint32_t bmU[ROWS * kCW], bmP[ROWS * kCW], bmD[ROWS * kCW];
    float4 xch[32];                       // exact: U rank -> value; fallback: producer lane -> value
    float4 mw[32];                        // per lane: merged corner weights (C+ spare lanes read the served lane's)
    uint32_t fpos[32];                    // per lane: cx0 | cx1 << 6 | cy0 << 12 | cy1 << 18 | contrib << 24
    uint16_t tbl[32];                     // rank -> window position r * COLS + c: exact U ranks / C+ plan
    uint8_t act[32];                      // active rank -> lane (h(r, A))
    uint4 lut[8];                         // BC1 per-index constants (bc1_lut_entry)
    uint8_t lop[ROWS * COLS];             // fallback: window position -> a lane that produced it (valid where bmD is set)
};
#ifndef CTF_REST_ROWS
#define CTF_REST_ROWS 32  // window rows of the wide-window kernel's bitmap (32 or 64)
#endif
// 64 rows in the second kernel: +1 % on config 4, -0.6 % on config 5 (more shared memory per
// warp), so 32 by default; the third kernel's 64 x 64 window takes the taller waves
using WideSmem = WideSmemT<CTF_REST_ROWS>;
using WideSmemBig = WideSmemT<64, 64>;

// exclusive prefix sum over the lanes (lane k holds the count of window row k)
// (shfl.up's in-range predicate guards the add: two instructions per step)
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, unsigned) {
    uint32_t s = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 u;\n\t"
                     "shfl.sync.up.b32 u|p, %0, %1, 0, 0xffffffff;\n\t@p add.u32 %0, %0, u;\n\t}"
                     : "+r"(s) : "r"(d));
    return s - v;
}
// rank of window texel (row r, column c) in a bitmap whose row r word is `word` and whose
// rows before r hold `base` set bits
__device__ __forceinline__ int bm_rank(uint32_t base, uint32_t word, int c) {
    return (int)base + __popc(word & ((1u << c) - 1u));
}
// the same over a CW-word row: the set bits of the row's words before c's word, then c's word
template <int CW>
__device__ __forceinline__ int win_rank(const uint32_t *bm, uint32_t base, int r, int c) {
    if constexpr (CW == 1) {
        return bm_rank(base, bm[r], c);
    } else {
        const uint32_t w0 = bm[2 * r], w1 = bm[2 * r + 1];
        return c < 32 ? bm_rank(base, w0, c) : bm_rank(base + (uint32_t)__popc(w0), w1, c - 32);
    }
}
// word index and bit of window texel (r, c)
template <int CW>
__device__ __forceinline__ int win_word(int r, int c) { return r * CW + (c >> 5); }
template <int CW>
__device__ __forceinline__ uint32_t win_bit(const uint32_t *bm, int r, int c) {
    return (bm[win_word<CW>(r, c)] >> (c & 31)) & 1u;
}
// row scan of a ROWS x (32 CW) bitmap: lane l holds row l (32 rows) or rows 2l, 2l + 1 (64
// rows); the row-major rank order is preserved
template <int ROWS, int CW>
struct RowScan {
    uint32_t be, c0, c, tot;   // set bits before the lane's first row; in that row; in the lane's rows; in the bitmap
};
// the counts only (tot: n of a fallback wave needs no ranks); row_scan_ranks adds the scan
template <int ROWS, int CW>
__device__ __forceinline__ RowScan<ROWS, CW> row_count(const uint32_t *bm, unsigned lane) {
    constexpr int WPL = ROWS / 32 * CW;   // words per lane
    RowScan<ROWS, CW> r;
    if constexpr (WPL == 1) {
        r.c = r.c0 = __popc(bm[lane]);
    } else if constexpr (WPL == 2) {
        const uint2 w = reinterpret_cast<const uint2 *>(bm)[lane];
        r.c0 = CW == 1 ? (uint32_t)__popc(w.x) : (uint32_t)(__popc(w.x) + __popc(w.y));
        r.c = (uint32_t)(__popc(w.x) + __popc(w.y));
    } else {
        const uint4 w = reinterpret_cast<const uint4 *>(bm)[lane];
        r.c0 = (uint32_t)(__popc(w.x) + __popc(w.y));
        r.c = r.c0 + (uint32_t)(__popc(w.z) + __popc(w.w));
    }
    r.be = 0u;
    r.tot = __reduce_add_sync(FULL, r.c);
    return r;
}
template <int ROWS, int CW>
__device__ __forceinline__ void row_scan_ranks(RowScan<ROWS, CW> &r, unsigned lane) { r.be = warp_excl_scan(r.c, lane); }
template <int ROWS, int CW>
__device__ __forceinline__ RowScan<ROWS, CW> row_scan(const uint32_t *bm, unsigned lane) {
    RowScan<ROWS, CW> r = row_count<ROWS, CW>(bm, lane);
    row_scan_ranks(r, lane);
    return r;
}
// set bits before row `row` (every lane participates)
template <int ROWS, int CW>
__device__ __forceinline__ uint32_t row_base(const RowScan<ROWS, CW> &rs, int row) {
    if constexpr (ROWS == 64) {
        const uint32_t be = __shfl_sync(FULL, rs.be, row >> 1), c0 = __shfl_sync(FULL, rs.c0, row >> 1);
        return be + ((row & 1) ? c0 : 0u);
    } else {
        return __shfl_sync(FULL, rs.be, row);
    }
}
// zero the lane's words of a bitmap
template <int ROWS, int CW>
__device__ __forceinline__ void bm_zero(uint32_t *bm, unsigned lane) {
    constexpr int WPL = ROWS / 32 * CW;
    if constexpr (WPL == 1) bm[lane] = 0u;
    else if constexpr (WPL == 2) reinterpret_cast<uint2 *>(bm)[lane] = make_uint2(0u, 0u);
    else reinterpret_cast<uint4 *>(bm)[lane] = make_uint4(0u, 0u, 0u, 0u);
}

// ROWS x COLS window: (32, 32) in the second kernel, (64, 64) in the third (BC1), which keeps
// the general (sort) path for AABBs beyond 64 x 64 only
template <bool DBG, int ROWS, int COLS = 32>
__device__ __forceinline__ LeanOut wide_wave(const KArgs &a, WideSmemT<ROWS, COLS> &ws, float2 uv, uint2 gr, bool inframe,
                                             int px, int py, uint32_t frame, bool force) {
    constexpr int CW = COLS / 32, LGC = COLS == 64 ? 6 : 5;
    const unsigned lane = lane_id(), lt = lanemask_lt();
    LeanOut o;
    o.color = make_float4(0.f, 0.f, 0.f, 0.f);
    o.prod = INVALID_ID;
    o.selbits = 0u;
    o.done = true;
    const bool active = inframe && !isnan(uv.x);
    const unsigned A = __ballot_sync(FULL, active);
    const int na = __popc(A);
    if (A == 0u) {   // empty wave: n = 0, zero colour
        o.rec = 1u << 26;
        return o;
    }
    // ---- a1: magnified class over the active lanes (R-20)
    bool mag_lane = true;
    if (a.grad) {
        const float rx = fma_f32_f16((unsigned short)(gr.x & 0xffffu), (unsigned short)(gr.x & 0xffffu),
                                     fma_f32_f16((unsigned short)(gr.x >> 16), (unsigned short)(gr.x >> 16), 0.0f));
        const float ry = fma_f32_f16((unsigned short)(gr.y & 0xffffu), (unsigned short)(gr.y & 0xffffu),
                                     fma_f32_f16((unsigned short)(gr.y >> 16), (unsigned short)(gr.y >> 16), 0.0f));
        mag_lane = !active || (rx <= 1.0f && ry <= 1.0f);
    }
    const bool wave_mag = a.grad != nullptr && __all_sync(FULL, mag_lane);
    // ---- a2: footprint; a3: AABB (inactive lanes do not count)
    const Foot f = footprint2(uv, a);
    const int minx = __reduce_min_sync(FULL, active ? f.xa : INT_MAX);
    const int miny = __reduce_min_sync(FULL, active ? f.ya : INT_MAX);
    const int bw = __reduce_max_sync(FULL, active ? f.xb : 0) - minx + 1;
    const int bh = __reduce_max_sync(FULL, active ? f.yb : 0) - miny + 1;
    if (bw > COLS || bh > ROWS) {   // wider than the bitmap: the next kernel (64 x 64 window / general path)
        o.done = false;
        o.rec = kSlowMark;
        return o;
    }
    const int cx0 = (f.xa - minx) & (COLS - 1), cx1 = (f.xb - minx) & (COLS - 1), cy0 = (f.ya - miny) & (ROWS - 1),
              cy1 = (f.yb - miny) & (ROWS - 1);
    const int ar = __popc(A & lt);   // active rank: lane = h(ar, A)
    bm_zero<ROWS, CW>(ws.bmU, lane);
    bm_zero<ROWS, CW>(ws.bmP, lane);
    bm_zero<ROWS, CW>(ws.bmD, lane);
    if (active) ws.act[ar] = (uint8_t)lane;
    __syncwarp();
    // ---- a3: the needed set U (every corner, zero weights included, R-4); no-return atomics:
    // the tables below are published by every lane that holds a texel (its rank and position do
    // not depend on the lane, so those lanes store the same value)
    if (active) {
        if constexpr (CW == 1) {
            const uint32_t pat = (1u << cx0) | (1u << cx1);
            atomicOr(&ws.bmU[cy0], pat);
            atomicOr(&ws.bmU[cy1], pat);
        } else {
            const int cx[2] = {cx0, cx1}, cy[2] = {cy0, cy1};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = cx[k & 1];
                atomicOr(&ws.bmU[win_word<CW>(cy[k >> 1], c)], 1u << (c & 31));
            }
        }
    }
    __syncwarp();
    RowScan<ROWS, CW> rsU = row_count<ROWS, CW>(ws.bmU, lane);   // ranks only for an exact wave
    const int n = (int)rsU.tot;
    // ---- a4: decide (List R-6; Box / Mask R-22)
    bool exact;
    if (a.variant == VAR_LIST) exact = n <= na;
    else if (a.variant == VAR_BOX) exact = bw * bh <= na;
    else {
        const int lim = a.variant == VAR_MASK16 ? 16 : 11;
        exact = bw <= lim && bh <= lim && n <= na;
    }
    exact = exact && !force;
    const uint32_t rec_base = ((uint32_t)na << 16) | ((uint32_t)wave_mag << 25) | ((uint32_t)(na < 32) << 26);
    if (exact) {
        int rho[4];
        bool produced;
        int qx, qy, evals;
        if (a.variant != VAR_BOX) {
            // ranks of the four corners; every lane publishes its corners' rank -> position
            row_scan_ranks(rsU, lane);
            const uint32_t b0 = row_base(rsU, cy0), b1 = row_base(rsU, cy1);
            rho[0] = win_rank<CW>(ws.bmU, b0, cy0, cx0);
            rho[1] = win_rank<CW>(ws.bmU, b0, cy0, cx1);
            rho[2] = win_rank<CW>(ws.bmU, b1, cy1, cx0);
            rho[3] = win_rank<CW>(ws.bmU, b1, cy1, cx1);
            if (active) {   // rank -> position (every lane holding the texel stores the same value)
                ws.tbl[rho[0]] = (uint16_t)((cy0 << LGC) | cx0);
                ws.tbl[rho[1]] = (uint16_t)((cy0 << LGC) | cx1);
                ws.tbl[rho[2]] = (uint16_t)((cy1 << LGC) | cx0);
                ws.tbl[rho[3]] = (uint16_t)((cy1 << LGC) | cx1);
            }
            __syncwarp();
            // ---- a5: active rank r < n produces U[r] (lane h(r, A))
            produced = active && ar < n;
            const uint32_t e = produced ? (uint32_t)ws.tbl[ar] : 0u;
            qx = minx + (int)(e & (COLS - 1));
            qy = miny + (int)(e >> LGC);
            evals = n;
        } else {
            // Box: active rank i < w*h produces AABB texel (i mod w, i div w) (LaneIdxToCoord,
            // P:1069-1076); a corner reads its AABB-local index (CoordToLaneIdx)
            const int area = bw * bh;
            produced = active && ar < area;
            const int jq = (int)__fdividef((float)ar + 0.5f, (float)bw);   // exact for bw <= 64, ar < 32
            qx = minx + (ar - jq * bw);
            qy = miny + (produced ? jq : 0);
            rho[0] = cy0 * bw + cx0;
            rho[1] = cy0 * bw + cx1;
            rho[2] = cy1 * bw + cx0;
            rho[3] = cy1 * bw + cx1;
            evals = area;
        }
        if (!produced) {
            qx = minx;
            qy = miny;
        }
        const float4 val = bc1_decode_unorm_lut(a.tex, qx, qy, ws.lut);
        if (produced) ws.xch[ar] = val;
        if (DBG) o.prod = produced ? (uint32_t)(qy * a.tex.W + qx) : INVALID_ID;
        __syncwarp();
        // ---- a6: gather by rank + blend (the exact-path chain, bit-identical to 4-tap)
        const float4 p[4] = {ws.xch[rho[0] & 31], ws.xch[rho[1] & 31], ws.xch[rho[2] & 31], ws.xch[rho[3] & 31]};
        if (active) o.color = blend4f(p, f.w);
        o.rec = rec_base | ((uint32_t)n << 8) | (uint32_t)evals;
        if (DBG && a.dbg_unread) {
            const unsigned bad = __reduce_add_sync(FULL, active ? (unsigned)(rho[0] >= evals) + (unsigned)(rho[1] >= evals) +
                                                                  (unsigned)(rho[2] >= evals) + (unsigned)(rho[3] >= evals)
                                                            : 0u);
            if (lane == 0 && bad) atomicAdd(a.dbg_unread, bad);
        }
        __syncwarp();
        return o;
    }
    // ---- a7 fallback: every active lane's STF corner (R-11, R-12)
    const int fb = a.fallback;
    const uint4 rn = philox4x32_10_rk(make_uint4((uint32_t)px, (uint32_t)(py + a.row0), frame, 0u), a.rk[0], a.rk[1]);
    const int ksel = stf_corner(f, rn);
    o.selbits = active ? (uint32_t)ksel : 0u;
    int qcx = (ksel & 1) ? cx1 : cx0, qcy = (ksel & 2) ? cy1 : cy0;
    bool produced = active;   // STF, WC, C: every active lane produces its STF texel
    const Merged m = merge_corners(f);   // this lane's distinct corners (R-14): its Eq. 1 and C+ candidates
    const unsigned C = contrib_bits(f, m);
    if (fb == FB_CPLUS) {
        // (1) the planned set P: STF texels deduplicated, ranked ascending (R-17)
        if (active) atomicOr(&ws.bmP[win_word<CW>(qcy, qcx)], 1u << (qcx & 31));
        // publish this lane's distinct corners (merged weights, R-14) for the spare lanes
        ws.mw[lane] = make_float4(m.dw[0], m.dw[1], m.dw[2], m.dw[3]);
        ws.fpos[lane] = (uint32_t)cx0 | ((uint32_t)cx1 << 6) | ((uint32_t)cy0 << 12) | ((uint32_t)cy1 << 18) | (C << 24);
        __syncwarp();
        const RowScan<ROWS, CW> rsP = row_scan<ROWS, CW>(ws.bmP, lane);
        const int np = (int)rsP.tot;
        const uint32_t bq = row_base(rsP, qcy);
        if (active) ws.tbl[win_rank<CW>(ws.bmP, bq, qcy, qcx)] = (uint16_t)((qcy << LGC) | qcx);   // same value per texel
        __syncwarp();
        produced = false;
        if (active) {
            if (ar < np) {   // (2) active rank i < n_p produces planned texel i (lane h(i, A))
                const uint32_t e = ws.tbl[ar];
                qcx = (int)(e & (COLS - 1));
                qcy = (int)(e >> LGC);
                produced = true;
            } else {         // (3) spare lane: serves lane l of Eq. 2 (R-18)
                const int l = ws.act[eq2_lane_rank(ar, np, na)];
                o.selbits |= (1u << 5) | ((uint32_t)l << 8);
                const uint32_t fp = ws.fpos[l];
                const float4 gw = ws.mw[l];
                const int gx0 = (int)(fp & 63u), gx1 = (int)((fp >> 6) & 63u), gy0 = (int)((fp >> 12) & 63u),
                          gy1 = (int)((fp >> 18) & 63u);
                unsigned PL;
                if constexpr (CW == 1) {
                    const uint32_t r0 = ws.bmP[gy0], r1 = ws.bmP[gy1];
                    PL = ((r0 >> gx0) & 1u) | (((r0 >> gx1) & 1u) << 1) | (((r1 >> gx0) & 1u) << 2) |
                         (((r1 >> gx1) & 1u) << 3);
                } else {
                    PL = win_bit<CW>(ws.bmP, gy0, gx0) | (win_bit<CW>(ws.bmP, gy0, gx1) << 1) |
                         (win_bit<CW>(ws.bmP, gy1, gx0) << 2) | (win_bit<CW>(ws.bmP, gy1, gx1) << 3);
                }
                // candidates: l's distinct nonzero-weight texels not planned, picked ~ merged
                // weight with u2 (the sums and the decision in fp32, in corner order, as cplus_pick)
                const unsigned cand = (fp >> 24) & ~PL & 15u;
                const float dw[4] = {gw.x, gw.y, gw.z, gw.w};
                float ps[4], wsum = 0.0f;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    wsum = __fadd_rn(wsum, ((cand >> k) & 1u) ? dw[k] : 0.0f);
                    ps[k] = wsum;
                }
                const float target = __fmul_rn(unit24(rn.z), wsum);
                const unsigned gt = cand & ((ps[0] > target ? 1u : 0u) | (ps[1] > target ? 2u : 0u) |
                                            (ps[2] > target ? 4u : 0u) | (ps[3] > target ? 8u : 0u));
                if (cand != 0u) {
                    const int pick = gt != 0u ? __ffs(gt) - 1 : 31 - __clz(cand);
                    qcx = (pick & 1) ? gx1 : gx0;
                    qcy = (pick & 2) ? gy1 : gy0;
                    produced = true;
                    o.selbits |= ((uint32_t)pick << 2) | (1u << 4);
                }
            }
        }
    }
    // ---- the single texel-production site (<= 1 evaluation per lane)
    const int qx = produced ? minx + qcx : minx, qy = produced ? miny + qcy : miny;
    const float4 val = bc1_decode_unorm_lut(a.tex, qx, qy, ws.lut);
    if (DBG) o.prod = produced ? (uint32_t)(qy * a.tex.W + qx) : INVALID_ID;
    const int evals = fb == FB_CPLUS ? __popc(__ballot_sync(FULL, produced)) : na;
    o.rec = rec_base | ((uint32_t)(n & 0xFF) << 8) | ((uint32_t)(PATH_FB_STF + fb) << 22) | (uint32_t)(evals & 0xFF);
    if (fb == FB_STF) {   // one-tap STF
        if (active) o.color = val;
        return o;
    }
    // ---- a7 finish: the produced set D (values in the producers' slots, one source lane per
    // texel), Eq. 1 / WC over the known corners
    const int pq = ((qy - miny) << LGC) | (qx - minx);   // window position; its word is pq >> 5
    uint32_t oD = 0u;
    if (produced) oD = atomicOr(&ws.bmD[pq >> 5], 1u << (pq & 31));
    if (produced) ws.xch[lane] = val;
    // the first producer of each texel publishes its lane (one writer per position)
    if (produced && !((oD >> (pq & 31)) & 1u)) ws.lop[pq] = (uint8_t)lane;
    __syncwarp();
    unsigned IN;
    if constexpr (CW == 1) {
        const uint32_t d0 = ws.bmD[cy0], d1 = ws.bmD[cy1];
        IN = ((d0 >> cx0) & 1u) | (((d0 >> cx1) & 1u) << 1) | (((d1 >> cx0) & 1u) << 2) | (((d1 >> cx1) & 1u) << 3);
    } else {
        IN = win_bit<CW>(ws.bmD, cy0, cx0) | (win_bit<CW>(ws.bmD, cy0, cx1) << 1) | (win_bit<CW>(ws.bmD, cy1, cx0) << 2) |
             (win_bit<CW>(ws.bmD, cy1, cx1) << 3);
    }
    const int p0 = cy0 << LGC, p2 = cy1 << LGC;
    if (fb == FB_WC) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 pv[4] = {(IN & 1u) ? ws.xch[ws.lop[p0 | cx0]] : z, (IN & 2u) ? ws.xch[ws.lop[p0 | cx1]] : z,
                              (IN & 4u) ? ws.xch[ws.lop[p2 | cx0]] : z, (IN & 8u) ? ws.xch[ws.lop[p2 | cx1]] : z};
        if (active) o.color = combine_eq1_mc<true>(f, m, C, IN, pv);
    } else {
        // C / C+: every slot holds a finite value (zeroed at kernel start), unknown corners get
        // coefficient 0, so the loads need no predicate
        const float4 pv[4] = {ws.xch[ws.lop[p0 | cx0] & 31], ws.xch[ws.lop[p0 | cx1] & 31],
                              ws.xch[ws.lop[p2 | cx0] & 31], ws.xch[ws.lop[p2 | cx1] & 31]};
        if (active) o.color = combine_eq1_coef(f, m, C, IN, pv);
    }
    __syncwarp();
    return o;
}


// GRAD: grad != NULL (magnified class); FORCE: CTF_FLAG_FORCE_FALLBACK (every live wave
// goes to the rest kernel) — compile-time, so the hot loop tests neither.
template <bool DBG, bool FORCE, int FMT>
constexpr bool kPaired = CTF_PAIR && !DBG && !FORCE && (FMT == FMT_BC1 || CTF_PAIR_MLP);
template <bool DBG>
static __device__ __noinline__ WaveOut general_wave_noinline(const KArgs &a, WarpSmem &s, float2 uv, uint2 gr,
                                                             bool active, unsigned A, int px, int py, uint32_t frame);
#ifndef CTF_MLP_WARPS
#define CTF_MLP_WARPS 8  // latent-MLP lean kernel: warps per CTA
#endif
#ifndef CTF_MLP_LEAN_MINB
#define CTF_MLP_LEAN_MINB (CTF_MLP_COLLAB_MINB * 8 / CTF_MLP_WARPS)  // latent-MLP lean kernel: CTAs per SM
#endif
// warps per CTA of the lean kernel: BC1 kWarps; latent MLP CTF_MLP_WARPS (its register budget)
template <int FMT>
__host__ __device__ constexpr int lean_warps() { return FMT == FMT_BC1 ? kWarps : CTF_MLP_WARPS; }
// the wide-window path out of line (the fused kernel keeps the lean loop's registers)
template <bool DBG>
static __device__ __noinline__ LeanOut wide_wave_noinline(const KArgs &a, WideSmemT<32> &ws, float2 uv, uint2 gr,
                                                          bool inframe, int px, int py, uint32_t frame, bool force) {
    return wide_wave<DBG, 32>(a, ws, uv, gr, inframe, px, py, frame, force);
}
// FUSED (BC1, small calls): the waves a run leaves are finished in the same kernel, right after
// the run (the wide-window path inline, the general path out of line) — one launch per call,
// no work lists, no counters; the larger register allocation costs occupancy, which small
// calls do not have to fill.
#ifndef CTF_FUSED_MINB
#define CTF_FUSED_MINB 6  // fused lean kernel: resident CTAs per SM (the lean loop's budget; the wide path is out of line)
#endif
#ifndef CTF_FUSED_MAX_WAVES
#define CTF_FUSED_MAX_WAVES 131072  // calls with at most this many waves run the fused kernel
#endif
#ifndef CTF_VBAND
#define CTF_VBAND 8  // wave-rows per band of the lean kernels' item order (1: row-major runs)
#endif
// work item rr of a frame -> (wave-row, run column).  Items run down bands of CTF_VBAND
// wave-rows first, so the consecutive items a CTA's warps take are vertically stacked runs:
// a BC1 block (4 x 4 texels, ~8-16 pixels tall when magnified) is shared by 2-4 of the CTA's
// wave-rows at about the same time, so its L2 round trip is paid once per SM (L1) instead of
// once per warp.  The last band of a frame holds the remaining nwy mod CTF_VBAND wave-rows.
__device__ __forceinline__ void run_coords(int rr, const KArgs &a, int &wy, int &wxc) {
    if constexpr (CTF_VBAND <= 1) {
        wy = rr / a.cpr;
        wxc = rr - wy * a.cpr;
    } else {
        const int bs = CTF_VBAND * a.cpr;
        const int band = rr / bs, q = rr - band * bs;
        const int h = min(CTF_VBAND, a.nwy - band * CTF_VBAND);
        wxc = h == CTF_VBAND ? q / CTF_VBAND : q / h;
        wy = band * CTF_VBAND + (q - wxc * h);
    }
}
template <bool DBG, bool GRAD, bool FORCE, int FMT, bool BOX = false, bool FUSED = false>
__global__ void __launch_bounds__(lean_warps<FMT>() * 32, FUSED ? CTF_FUSED_MINB
                                                     : FMT == FMT_BC1 ? (kPaired<DBG, FORCE, FMT> ? CTF_PAIR_MINB : CTF_FAST_MINB)
                                                                      : CTF_MLP_LEAN_MINB)
    ctf_collab_lean_kernel(const __grid_constant__ KArgs a, const typename WeightsOf<FMT>::type mw) {
    static_assert(!FUSED || FMT == FMT_BC1, "the fused kernel is BC1-only");
    constexpr int kLW = lean_warps<FMT>();
    constexpr bool PAIR = kPaired<DBG, FORCE, FMT>;
    using SmemT = std::conditional_t<PAIR, PairSmem, FastSmem>;
    __shared__ SmemT fsm[kLW];
    __shared__ WideSmemT<32> wsm[FUSED ? kLW : 1];
    __shared__ WarpSmem gsm[FUSED ? kLW : 1];
    extern __shared__ __align__(16) unsigned char dyn_smem[];   // latent MLP: TcWeights + per-warp TcScratch
    const unsigned lane = lane_id(), warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);   // provably warp-uniform (no divergence guards)
    SmemT &fs = fsm[warp];
    MlpCtx mc{nullptr, nullptr, nullptr, dyn_smem, warp};
    WideSmemT<32> &ws = wsm[FUSED ? warp : 0];
    if constexpr (FMT == FMT_BC1) {
        if (lane < 8) fs.lut[lane] = bc1_lut_entry(lane);
        if (FUSED && lane < 8) ws.lut[lane] = bc1_lut_entry(lane);
        if (FUSED) ws.xch[lane] = make_float4(0.f, 0.f, 0.f, 0.f);   // finite slots (combine_eq1_coef)
        __syncwarp();
    }
    __shared__ unsigned s_next;   // latent MLP: the CTA's warps claim its items dynamically
    if constexpr (FMT != FMT_BC1) {
        TcWeights &tw = *reinterpret_cast<TcWeights *>(dyn_smem);
        fill_tc_weights(mw, tw);
        mc.tw = &tw;
        mc.tsc = &reinterpret_cast<TcScratch *>(dyn_smem + sizeof(TcWeights))[warp];
        if (threadIdx.x == 0) s_next = kLW;
        __syncthreads();
    }
    // programmatic dependent launch: a one-wave grid lets the next kernel on the stream launch
    // now (its CTAs take the free slots and wait for this grid); every grid waits for the
    // previous kernel's results before its first global access (the prologue above overlaps it)
    if (a.flags & FLAG_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lx = (int)(lane & 7), ly = (int)(lane >> 3);
    const unsigned per_warp = a.ipc / kLW;
    for (unsigned k = warp;;) {
        // BC1: warp (b, w) takes items b*kLW + w + j*gridDim.x*kLW (static); latent MLP:
        // CTA b owns items b + k*gridDim.x and its warps claim k from a shared counter
        // (decode cost varies with n: dynamic claims balance the warps of a CTA)
        const unsigned c = FMT == FMT_BC1 ? (blockIdx.x * kLW + (k % kLW)) + (k / kLW) * gridDim.x * kLW
                                          : blockIdx.x + k * gridDim.x;
        if ((FMT == FMT_BC1 ? k / kLW >= per_warp : k >= a.ipc) || c >= a.nchunks) break;
        if constexpr (FMT == FMT_BC1) {
            k += kLW;
        } else {
            unsigned nx = 0u;
            if (lane == 0) nx = atomicAdd(&s_next, 1u);
            k = __shfl_sync(FULL, nx, 0);
        }
        const int fr = (int)(c / (unsigned)a.cpf);
        const int rr = (int)(c - (unsigned)fr * (unsigned)a.cpf);
        int wy, wxc;
        run_coords(rr, a, wy, wxc);
        // run wxc of the wave-row: lengths differ by at most one wave (<= chunk)
        const int wx0 = (int)udiv_magic((unsigned)(wxc * a.nwx), a.cpr_m, a.cpr_s);
        const int wx1 = (int)udiv_magic((unsigned)((wxc + 1) * a.nwx), a.cpr_m, a.cpr_s);
        const int py = wy * 4 + ly;
        const bool rowok = py < a.Hf;
        const bool rowok_all = wy * 4 + 4 <= a.Hf;   // warp-uniform: all 4 rows in the frame
        const uint32_t frame = a.frame_index + (uint32_t)fr;
        const unsigned w0 = (unsigned)fr * (unsigned)a.wpf + (unsigned)(wy * a.nwx + wx0);
        unsigned pix = (unsigned)fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)(wx0 * 8 + lx);
        int px = wx0 * 8 + lx;
        constexpr bool has_grad = GRAD;
        float2 uv_n = make_float2(__int_as_float(0x7fc00000), 0.f);
        uint2 gr_n = make_uint2(0u, 0u);
        ld_stream_f2_if(uv_n, a.uv + pix, rowok & (px < a.Wf));
        ld_stream_u2_if(gr_n, a.grad + pix, rowok & (px < a.Wf) & has_grad);
        // interior runs (every pixel of the run in the frame, the common case) drop the
        // per-wave bounds predicates: the loop is instantiated twice
        uint32_t myrec = 0u;
        auto run = [&](auto interior_tag) {
          constexpr bool INTERIOR = decltype(interior_tag)::value;
          if constexpr (INTERIOR && PAIR) {
            // pairs (A, B) = waves (wx, wx + 1); A's next load is issued after A's front,
            // B's after B's front, so each covers about one pair of work
            const unsigned lt_mask = lanemask_lt();
            const uint32_t cpk = push_codes(lane);
            float2 uv_b = make_float2(__int_as_float(0x7fc00000), 0.f);
            uint2 gr_b = make_uint2(0u, 0u);
            ld_stream_f2_if(uv_b, a.uv + (pix + 8u), wx0 + 1 < wx1);
            ld_stream_u2_if(gr_b, a.grad + (pix + 8u), (wx0 + 1 < wx1) & has_grad);
            for (int wx = wx0; wx < wx1; wx += 2, pix += 16u) {
              const bool hasB = wx + 1 < wx1;
              const PairFront fa = pair_front<GRAD, FMT, SmemT, BOX>(a, fs, uv_n, gr_n, 0, fs.bit_of_rank, lane, lt_mask, cpk);
              ld_stream_f2_if(uv_n, a.uv + (pix + 16u), wx + 2 < wx1);
              ld_stream_u2_if(gr_n, a.grad + (pix + 16u), (wx + 2 < wx1) & has_grad);
              PairFront fb;
              fb.n = 0;
              fb.rec = 0u;
              __syncwarp();   // A's push-table writes (all of them, also a rejected A's) before B's
              if (hasB) fb = pair_front<GRAD, FMT, SmemT, BOX>(a, fs, uv_b, gr_b, fa.n, fs.bit_of_rank, lane, lt_mask, cpk);
              ld_stream_f2_if(uv_b, a.uv + (pix + 24u), wx + 3 < wx1);
              ld_stream_u2_if(gr_b, a.grad + (pix + 24u), (wx + 3 < wx1) & has_grad);
              __syncwarp();   // bit_of_rank written; the previous pair's xch reads are done
              pair_decode<FMT>(a, fs, fs.bit_of_rank, fa, fb, lane, mc);
              __syncwarp();
              pair_back(a, fs, fa, pix);
              if (hasB) pair_back(a, fs, fb, pix + 8u);
              if (lane == (unsigned)(wx - wx0)) myrec = fa.rec;
              if (lane == (unsigned)(wx + 1 - wx0)) myrec = hasB ? fb.rec : myrec;
            }
          } else {
          for (int wx = wx0; wx < wx1; ++wx, pix += 8u, px += 8) {
            const bool inframe = INTERIOR || (rowok & (px < a.Wf));
            const float2 uv = uv_n;
            const uint2 gr = gr_n;
            const bool pf = INTERIOR ? (wx + 1 < wx1) : ((wx + 1 < wx1) & rowok & (px + 8 < a.Wf));
            ld_stream_f2_if(uv_n, a.uv + (pix + 8u), pf);
            ld_stream_u2_if(gr_n, a.grad + (pix + 8u), pf & has_grad);
            __syncwarp();  // the previous wave's shared-memory reads are done

            const bool active = inframe && !isnan(uv.x);
            const unsigned A = __ballot_sync(FULL, active);
            uint32_t rec;
            if (!FORCE && A == FULL) {
                const LeanOut o = lean_wave<DBG, FMT, SmemT, BOX>(a, fs, fs.lut, mc, uv, gr, GRAD);
                rec = o.rec;
                if (o.done) {
                    st_stream_f4(a.out + pix, o.color);
                    if (DBG) {
                        if (a.dbg_pid) a.dbg_pid[pix] = o.prod;
                        if (a.dbg_sel) a.dbg_sel[pix] = 0u;
                    }
                }
            } else if (A == 0u) {   // empty wave: partial, n = 0, zero colour
                rec = 1u << 26;
                if (inframe) st_stream_f4(a.out + pix, make_float4(0.f, 0.f, 0.f, 0.f));
                if (DBG && inframe) {
                    if (a.dbg_pid) a.dbg_pid[pix] = INVALID_ID;
                    if (a.dbg_sel) a.dbg_sel[pix] = 0u;
                }
            } else {
                // partial (or, FORCE, any live) wave: the wide-window / third kernel (BC1), the general kernel
                if constexpr (FMT == FMT_BC1) rec = bc1_rest_mark(footprint2(uv, a), active);
                else rec = kSlowMark;
            }
            if (lane == (unsigned)(wx - wx0)) myrec = rec;
          }
          }
        };
        if (rowok_all && wx1 * 8 <= a.Wf) run(std::true_type{});
        else run(std::false_type{});
        const bool inrun = lane < (unsigned)(wx1 - wx0);
        if constexpr (FUSED) {
            // finish the run's marked waves here: the wide-window path, else (AABB wider than
            // 32 x 32) the general path out of line
            unsigned todo = __ballot_sync(FULL, inrun && (myrec == kFbMark || myrec == kSlowMark));
            while (todo) {
                const int b = __ffs(todo) - 1;
                todo &= todo - 1u;
                const int pxb = (wx0 + b) * 8 + lx;
                const bool inf = rowok & (pxb < a.Wf);
                const unsigned pixb = (unsigned)fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)pxb;
                float2 uvb = make_float2(__int_as_float(0x7fc00000), 0.f);
                uint2 grb = make_uint2(0u, 0u);
                ld_stream_f2_if(uvb, a.uv + pixb, inf);
                ld_stream_u2_if(grb, a.grad + pixb, inf & has_grad);
                __syncwarp();
                LeanOut o = wide_wave_noinline<DBG>(a, ws, uvb, grb, inf, pxb, py, frame, FORCE);
                if (!o.done) {
                    const bool act = inf && !isnan(uvb.x);
                    const WaveOut go = general_wave_noinline<DBG>(a, gsm[warp], uvb, grb, act, __ballot_sync(FULL, act),
                                                                  pxb, py, frame);
                    o.color = go.color;
                    o.rec = go.rec;
                    o.prod = go.prod;
                    o.selbits = go.selbits;
                }
                if (inf) st_stream_f4(a.out + pixb, o.color);
                if (DBG && inf) {
                    if (a.dbg_pid) a.dbg_pid[pixb] = o.prod;
                    if (a.dbg_sel) a.dbg_sel[pixb] = o.selbits;
                }
                if (lane == (unsigned)b) myrec = o.rec;
            }
        }
        if (inrun) a.rec[w0 + lane] = myrec;
        // this run's fallback / general waves (lane = wave of the run)
        const unsigned mfb = __ballot_sync(FULL, inrun && myrec == kFbMark);
        const unsigned msl = __ballot_sync(FULL, inrun && myrec == kSlowMark);
        if (a.lists && (mfb | msl)) {   // append the run's marked waves to the work lists (predicated)
            const unsigned b0 = __shfl_sync(FULL, atom_add_if(a.lcnt + 0, (unsigned)__popc(mfb), lane == 0 && mfb), 0);
            const unsigned b1 = __shfl_sync(FULL, atom_add_if(a.lcnt + 1, (unsigned)__popc(msl), lane == 0 && msl), 0);
            const unsigned lt = lanemask_lt();
            st_u32_if(a.lists + b0 + __popc(mfb & lt), w0 + lane, (mfb >> lane) & 1u);
            st_u32_if(a.lists + a.nrec + b1 + __popc(msl & lt), w0 + lane, (msl >> lane) & 1u);
        }
    }
}

// ---- latent MLP: CTA-level tensor-core (tcgen05) decode of the lean waves' texels
#ifndef CTF_TC05
#define CTF_TC05 0  // 1: latent-MLP COLLAB release path on the CTA-level tcgen05 kernel (measured slower
                    // than the one-warp mma.sync path, profiles/r02/tc05_evaluation.md)
#endif
#ifndef CTF_TC05_MINB
#define CTF_TC05_MINB 3  // resident CTAs (8 warps each) per SM
#endif
#include "ctf_mlp_tc05.cuh"

// Second / third pass over the marked waves.  FALLBACK: the kFbMark waves through the lean
// fallback (fb_wave) — and, with CTF_REST_MERGED, the kSlowMark waves through the general
// path out of line; else (third kernel) the kSlowMark waves through the general path.
// Warps stride over groups of 32 records (one coalesced 128-B load + ballot each).
#ifndef CTF_REST_MINB
#define CTF_REST_MINB 3  // general kernel: resident CTAs per SM (80 registers: the general path fits)
#endif
#ifndef CTF_FB_MINB
#define CTF_FB_MINB 4  // fallback kernel: resident CTAs per SM (64 registers)
#endif
constexpr int kScanGroups = 8;   // record groups loaded per warp step in the rest kernels
#ifndef CTF_REST_BIG
#define CTF_REST_BIG 1  // 1: the third kernel (BC1) tries the 64 x 64 bitmap window before the sort-based general path
#endif
#ifndef CTF_REST_MERGED
#define CTF_REST_MERGED 0  // 1: the fallback kernel also runs the general path (out of line); no third kernel
#endif
// the general path for one wave; OUT_OF_LINE keeps its register demand out of the
// fallback kernel's allocation (it spills instead; those waves are rare)
template <bool DBG>
static __device__ __noinline__ WaveOut general_wave_noinline(const KArgs &a, WarpSmem &s, float2 uv, uint2 gr,
                                                             bool active, unsigned A, int px, int py, uint32_t frame) {
    const MlpCtx mc{nullptr, nullptr, nullptr, nullptr, 0u};
    return wave_general<FMT_BC1, MODE_COLLAB, DBG>(a, NoWeights{}, s, mc, uv, gr, active, A, __popc(A), px, py, frame);
}
template <bool DBG, bool OUT_OF_LINE>
__device__ __forceinline__ WaveOut general_wave(const KArgs &a, WarpSmem &s, float2 uv, uint2 gr, bool active,
                                                unsigned A, int px, int py, uint32_t frame) {
    if constexpr (OUT_OF_LINE) {
        return general_wave_noinline<DBG>(a, s, uv, gr, active, A, px, py, frame);
    } else {
        const MlpCtx mc{nullptr, nullptr, nullptr, nullptr, 0u};
        return wave_general<FMT_BC1, MODE_COLLAB, DBG>(a, NoWeights{}, s, mc, uv, gr, active, A, __popc(A), px, py,
                                                       frame);
    }
}
template <bool DBG, bool FALLBACK, int FMT>
__global__ void __launch_bounds__(kWarps * 32, FALLBACK ? CTF_FB_MINB : (FMT == FMT_BC1 ? CTF_REST_MINB : CTF_MLP_COLLAB_MINB))
    ctf_collab_rest_kernel(const __grid_constant__ KArgs a, unsigned nrec, const typename WeightsOf<FMT>::type mw) {
    static_assert(FMT == FMT_BC1 || !FALLBACK, "no lean fallback for the latent-MLP format");
    // launched as a programmatic dependent of the previous pass: wait for its results.  CONC
    // (BC1, the lean kernel routes by AABB): the third kernel runs right after the lean kernel and
    // lets the wide-window kernel launch at once; the wide-window kernel reads only the lean
    // kernel's results (complete and visible: every third-kernel CTA triggered after its own
    // wait) and waits for the third kernel before it completes, so the call's stream order holds
    constexpr bool CONC = FMT == FMT_BC1 && CTF_REST_CONCURRENT && !CTF_REST_MERGED;
    struct EndWait {
        bool on;
        __device__ ~EndWait() {
            if (on) asm volatile("griddepcontrol.wait;" ::: "memory");
        }
    } end_wait{CONC && FALLBACK};
    if (!(CONC && FALLBACK)) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (CONC && !FALLBACK) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (a.lists && a.lcnt[FALLBACK ? 0 : 1] == 0u) return;   // empty work list (same value in every thread)
    // BIG: the third kernel (BC1) runs the 64 x 64 window first; the sort-based general path
    // only takes AABBs beyond it
    constexpr bool BIG = !FALLBACK && FMT == FMT_BC1 && CTF_REST_BIG;
    __shared__ WarpSmem smem[(FALLBACK && !CTF_REST_MERGED) ? 1 : kWarps];
    __shared__ WideSmem fsm[FALLBACK ? kWarps : 1];
    extern __shared__ __align__(16) unsigned char dyn_smem[];   // latent MLP: TcWeights + per-warp TcScratch
    const unsigned lane = lane_id(), warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);   // provably warp-uniform (no divergence guards)
    WarpSmem &s = smem[(FALLBACK && !CTF_REST_MERGED) ? 0 : warp];
    WideSmem &fs = fsm[FALLBACK ? warp : 0];
    MlpCtx mc{nullptr, nullptr, nullptr, dyn_smem, warp};
    // the 64 x 64 windows live in dynamic shared memory (kWarps x ~7 KB)
    WideSmemBig &fb = reinterpret_cast<WideSmemBig *>(dyn_smem)[BIG ? warp : 0];
    if (FALLBACK) {
        if (lane < 8) fs.lut[lane] = bc1_lut_entry(lane);
        fs.xch[lane] = make_float4(0.f, 0.f, 0.f, 0.f);   // finite values in every slot (combine_eq1_coef)
        __syncwarp();
    }
    if (BIG) {
        if (lane < 8) fb.lut[lane] = bc1_lut_entry(lane);
        fb.xch[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
    }
    if constexpr (FMT != FMT_BC1) {
        TcWeights &tw = *reinterpret_cast<TcWeights *>(dyn_smem);
        fill_tc_weights(mw, tw);
        mc.tw = &tw;
        mc.tsc = &reinterpret_cast<TcScratch *>(dyn_smem + sizeof(TcWeights))[warp];
        __syncthreads();
    }
    const int lx = (int)(lane & 7), ly = (int)(lane >> 3);
    // one marked wave: lean fallback (FALLBACK) or the general path
    auto process = [&](unsigned wi, float2 uv, uint2 gr, unsigned fr, int px, int py, bool inframe, unsigned pix) {
        __syncwarp();
        const bool active = inframe && !isnan(uv.x);
        const unsigned A = __ballot_sync(FULL, active);
        const uint32_t frame = a.frame_index + fr;
        LeanOut o;
        o.done = false;
        if (FALLBACK) o = wide_wave<DBG, CTF_REST_ROWS>(a, fs, uv, gr, inframe, px, py, frame, (a.flags & FLAG_FORCE_FALLBACK) != 0u);
        else if constexpr (BIG) o = wide_wave<DBG, 64, 64>(a, fb, uv, gr, inframe, px, py, frame, (a.flags & FLAG_FORCE_FALLBACK) != 0u);
        if (!o.done) {
            if (FALLBACK && !CTF_REST_MERGED) {   // AABB wider than 32 x 32 texels: general kernel
                if (lane == 0) {
                    a.rec[wi] = kSlowMark;
                    if (a.lists) a.lists[a.nrec + atomicAdd(a.lcnt + 1, 1u)] = wi;
                }
                return;
            }
            WaveOut go;
            if constexpr (FMT == FMT_BC1)
                go = general_wave<DBG, FALLBACK && CTF_REST_MERGED>(a, s, uv, gr, active, A, px, py, frame);
            else
                go = wave_general<FMT, MODE_COLLAB, DBG>(a, mw, s, mc, uv, gr, active, A, __popc(A), px, py, frame);
            o.color = go.color;
            o.rec = go.rec;
            o.prod = go.prod;
            o.selbits = go.selbits;
        }
        if (inframe) st_stream_f4(a.out + pix, o.color);
        if (DBG && inframe) {
            if (a.dbg_pid) a.dbg_pid[pix] = o.prod;
            if (a.dbg_sel) a.dbg_sel[pix] = o.selbits;
        }
        if (lane == 0) a.rec[wi] = o.rec;
    };
    if (a.lists) {
        // ---- work-list mode: the waves the lean kernel appended, one per warp step
        // (balanced over the whole grid), the next one's inputs loaded ahead
        const unsigned n = __shfl_sync(FULL, a.lcnt[FALLBACK ? 0 : 1], 0);   // provably uniform
        const uint32_t *L = a.lists + (FALLBACK ? 0u : a.nrec);
        const unsigned tw = gridDim.x * kWarps;
        unsigned i = blockIdx.x * kWarps + warp;
        if (i >= n) return;
        auto fetch_wi = [&](unsigned wi, float2 &uv, uint2 &gr, unsigned &fr, int &px, int &py, bool &inframe,
                            unsigned &pix) {
            fr = udiv_magic(wi, a.wpf_m, a.wpf_s);
            const unsigned rem = wi - fr * (unsigned)a.wpf;
            const int wy = (int)udiv_magic(rem, a.nwx_m, a.nwx_s), wx = (int)rem - wy * a.nwx;
            px = wx * 8 + lx;
            py = wy * 4 + ly;
            inframe = px < a.Wf && py < a.Hf;
            pix = fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)px;
            uv = make_float2(__int_as_float(0x7fc00000), 0.f);
            gr = make_uint2(0u, 0u);
            ld_stream_f2_if(uv, a.uv + pix, inframe);
            ld_stream_u2_if(gr, a.grad + pix, inframe & (a.grad != nullptr));
        };
        // list entries are loaded two waves ahead (the entry's load latency is not on the
        // critical path of the next wave's input fetch), inputs one wave ahead
        unsigned wi_n = __shfl_sync(FULL, L[i], 0), fr_n, pix_n;
        unsigned wi_nn = 0u;
        ld_u32_if(wi_nn, L + (i + tw), lane == 0 && i + tw < n);
        float2 uv_n;
        uint2 gr_n;
        int px_n, py_n;
        bool in_n;
        fetch_wi(wi_n, uv_n, gr_n, fr_n, px_n, py_n, in_n, pix_n);
        for (; i < n; i += tw) {
            const unsigned wi = wi_n, fr = fr_n, pix = pix_n;
            const float2 uv = uv_n;
            const uint2 gr = gr_n;
            const int px = px_n, py = py_n;
            const bool inframe = in_n;
            if (i + tw < n) {
                wi_n = __shfl_sync(FULL, wi_nn, 0);
                ld_u32_if(wi_nn, L + (i + 2 * tw), lane == 0 && i + 2 * tw < n);
                fetch_wi(wi_n, uv_n, gr_n, fr_n, px_n, py_n, in_n, pix_n);
            }
            process(wi, uv, gr, fr, px, py, inframe, pix);
        }
        return;
    }
    // ---- record-scan mode: groups of 32 records (marked waves cluster: fine groups balance better), kScanGroups
    // groups per warp step loaded together (the scan is latency-bound where nothing is marked)
    const unsigned ngroups = (nrec + 31u) / 32u, gwarps = gridDim.x * kWarps;
    for (unsigned g0 = blockIdx.x * kWarps + warp; g0 < ngroups; g0 += kScanGroups * gwarps) {
      uint32_t rs[kScanGroups];
#pragma unroll
      for (int j = 0; j < kScanGroups; ++j) {   // volatile: all loads issue before the first use
          const unsigned gj = g0 + (unsigned)j * gwarps;
          rs[j] = 0u;
          ld_u32_if(rs[j], a.rec + gj * 32u + lane, gj < ngroups && gj * 32u + lane < nrec);
      }
#pragma unroll 1
      for (int j = 0; j < kScanGroups; ++j) {
        const unsigned g = g0 + (unsigned)j * gwarps;
        const uint32_t r = rs[j];
        unsigned todo = FALLBACK ? __ballot_sync(FULL, r == kFbMark || (CTF_REST_MERGED && r == kSlowMark))
                                 : __ballot_sync(FULL, r == kSlowMark);
        if (!todo) continue;
        const unsigned wi0 = g * 32u;
        // wave coordinates of the group's first record (one division per group), then
        // of record wi0 + b by carrying b across wave-rows and frames
        const unsigned fr0 = wi0 / (unsigned)a.wpf, rem0 = wi0 - fr0 * (unsigned)a.wpf;
        const int wy0 = (int)(rem0 / (unsigned)a.nwx), wx00 = (int)rem0 - wy0 * a.nwx;
        auto locate = [&](unsigned b, unsigned &fr, int &wy, int &wx) {
            fr = fr0;
            wy = wy0;
            wx = wx00 + (int)b;
            while (wx >= a.nwx) {
                wx -= a.nwx;
                if (++wy == a.nwy) { wy = 0; ++fr; }
            }
        };
        // the next marked wave's inputs are loaded before the current one is processed
        auto fetch = [&](unsigned b, float2 &uv, uint2 &gr, unsigned &fr, int &px, int &py, bool &inframe,
                         unsigned &pix) {
            int wy, wx;
            locate(b, fr, wy, wx);
            px = wx * 8 + lx;
            py = wy * 4 + ly;
            inframe = px < a.Wf && py < a.Hf;
            pix = fr * a.fpx + (unsigned)py * (unsigned)a.Wf + (unsigned)px;
            uv = make_float2(__int_as_float(0x7fc00000), 0.f);
            gr = make_uint2(0u, 0u);
            ld_stream_f2_if(uv, a.uv + pix, inframe);
            ld_stream_u2_if(gr, a.grad + pix, inframe & (a.grad != nullptr));
        };
        float2 uv_n;
        uint2 gr_n;
        unsigned fr_n, pix_n;
        int px_n, py_n;
        bool in_n;
        unsigned b_n = (unsigned)(__ffs(todo) - 1);
        fetch(b_n, uv_n, gr_n, fr_n, px_n, py_n, in_n, pix_n);
        while (todo) {
            const unsigned wi = wi0 + b_n;
            const float2 uv = uv_n;
            const uint2 gr = gr_n;
            const unsigned fr = fr_n, pix = pix_n;
            const int px = px_n, py = py_n;
            const bool inframe = in_n;
            todo &= todo - 1u;
            if (todo) {
                b_n = (unsigned)(__ffs(todo) - 1);
                fetch(b_n, uv_n, gr_n, fr_n, px_n, py_n, in_n, pix_n);
            }
            process(wi, uv, gr, fr, px, py, inframe, pix);
        }
      }
    }
}

template <int FMT, int MODE, bool DBG>
static cudaError_t launch_one(KArgs k, const typename WeightsOf<FMT>::type &mw, cudaStream_t stream) {
    auto kern = ctf_filter_kernel<FMT, MODE, DBG>;
    int dev = 0, sms = 0, per_sm = 0;
#if CTF_MLP_TC
    const size_t dyn = (FMT == FMT_MLP && MODE == MODE_COLLAB) ? sizeof(TcWeights) + kWarps * sizeof(TcScratch) : 0;
#else
    const size_t dyn = (FMT == FMT_MLP && MODE == MODE_COLLAB) ? kWarps * sizeof(MlpBatchSmem) : 0;
#endif
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    if (dyn > 0) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
        // ask for a shared-memory carveout that holds the register-limited number of CTAs
        // (the default config can be too small for two 58 KB CTAs, halving occupancy)
        int max_smem = 0, regs_ctas = 0;
        e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        if (e != cudaSuccess) return e;
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        regs_ctas = 65536 / (fa.numRegs * kWarps * 32);
        const size_t per_cta = dyn + fa.sharedSizeBytes + 1024;  // + the driver's reserved 1 KB
        const int pct = (int)((100 * per_cta * (size_t)(regs_ctas > 0 ? regs_ctas : 1) + max_smem - 1) / max_smem);
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
        if (e != cudaSuccess) return e;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, dyn);
    if (e != cudaSuccess) return e;
    // items per CTA.  BC1: ipc / kWarps items per warp, 1..4, about CTF_BC1_ROUNDS CTAs
    // per resident slot (small batches keep the tail short; 4 per warp bounds the number
    // of CTAs of a 64-frame batch).  Latent-MLP: one CTA per slot.
    const long long slots = (long long)sms * (per_sm > 0 ? per_sm : 1);
    long long ipc;
    if (FMT == FMT_BC1) {
        long long ipw = ((long long)k.nchunks + slots * kWarps * CTF_BC1_ROUNDS / 2) / (slots * kWarps * CTF_BC1_ROUNDS);
        ipw = ipw < 1 ? 1 : ipw > CTF_BC1_MAX_IPW ? CTF_BC1_MAX_IPW : ipw;
        ipc = ipw * kWarps;
    } else {
        ipc = ((long long)k.nchunks + slots - 1) / slots;
        if (ipc < 1) ipc = 1;
    }
    k.ipc = (unsigned)ipc;
    long long grid = ((long long)k.nchunks + ipc - 1) / ipc;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kWarps * 32, dyn, stream>>>(k, mw);
    return cudaGetLastError();
}

#ifndef CTF_FAST
#define CTF_FAST 1  // COLLAB List runs the lean kernels (0: the general kernel, for A/B timing)
#endif
// dynamic shared memory of the latent-MLP kernels (tensor-core weights + per-warp scratch),
// with a carveout that holds the register-limited number of CTAs
template <typename Kern>
static cudaError_t mlp_smem_setup(Kern kern, size_t dyn, int dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    int max_smem = 0;
    e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const int regs_ctas = 65536 / (fa.numRegs * kWarps * 32);
    const size_t per_cta = dyn + fa.sharedSizeBytes + 1024;   // + the driver's reserved 1 KB
    const int pct = (int)((100 * per_cta * (size_t)(regs_ctas > 0 ? regs_ctas : 1) + max_smem - 1) / max_smem);
    return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
}

// The lean COLLAB (List) pass: the lean exact kernel, then (BC1) the lean fallback kernel
// and the general kernel over the waves it marked / appended to the work lists; (latent
// MLP) the general kernel over them.  Same work split as the general BC1 kernel.
// the lean exact kernel over k's frames
// one launch per call (the fused kernel) for BC1 calls of at most CTF_FUSED_MAX_WAVES waves,
// unless the caller asks for separate passes (FLAG_SEPARATE_PASSES; results are identical)
template <int FMT>
static bool use_fused(const KArgs &k) {
    return FMT == FMT_BC1 && k.nrec <= (unsigned)CTF_FUSED_MAX_WAVES && !(k.flags & FLAG_SEPARATE_PASSES);
}
template <int FMT, bool DBG, bool FUSED>
static auto lean_kernel_for(const KArgs &k) {
    constexpr bool F = FUSED && FMT == FMT_BC1;
    const bool grad = k.grad != nullptr, force = (k.flags & FLAG_FORCE_FALLBACK) != 0;
    auto kern = grad ? (force ? ctf_collab_lean_kernel<DBG, true, true, FMT, false, F>
                              : ctf_collab_lean_kernel<DBG, true, false, FMT, false, F>)
                     : (force ? ctf_collab_lean_kernel<DBG, false, true, FMT, false, F>
                              : ctf_collab_lean_kernel<DBG, false, false, FMT, false, F>);
    if (k.variant == VAR_BOX && !force)   // Box (forced: every live wave leaves the lean path anyway)
        kern = grad ? ctf_collab_lean_kernel<DBG, true, false, FMT, true, F>
                    : ctf_collab_lean_kernel<DBG, false, false, FMT, true, F>;
    return kern;
}
template <int FMT, bool DBG>
static cudaError_t launch_lean(KArgs &k, const typename WeightsOf<FMT>::type &mw, int dev, int sms,
                               cudaStream_t stream) {
    if constexpr (FMT == FMT_MLP && !DBG && CTF_TC05) {
        if (!(k.flags & FLAG_FORCE_FALLBACK)) {   // the CTA-level tensor-core path (ctf_mlp_tc05.cuh)
            const bool grad = k.grad != nullptr, box = k.variant == VAR_BOX;
            auto kern = grad ? (box ? ctf_mlp_tc05_kernel<true, true> : ctf_mlp_tc05_kernel<true, false>)
                             : (box ? ctf_mlp_tc05_kernel<false, true> : ctf_mlp_tc05_kernel<false, false>);
            const size_t dyn = sizeof(tc05::CtaSmem) + 1024;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            if (e != cudaSuccess) return e;
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            if (e != cudaSuccess) return e;
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tc05::kWarpsT * 32, dyn);
            if (e != cudaSuccess) return e;
            if (getenv("CTF_DEBUG_OCC")) {
                cudaFuncAttributes fa;
                cudaFuncGetAttributes(&fa, kern);
                fprintf(stderr, "tc05: per_sm %d dyn %zu nchunks %u sms %d | static %zu maxdyn %d regs %d maxthr %d local %zu\n",
                        per_sm, dyn, k.nchunks, sms, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.numRegs,
                        fa.maxThreadsPerBlock, fa.localSizeBytes);
            }
            // the occupancy API reports one CTA per SM for kernels that allocate tensor memory; each
            // CTA here holds 32 TMEM columns (of 512), so CTF_TC05_MINB CTAs fit (registers and
            // shared memory were sized for it)
            if (per_sm < CTF_TC05_MINB) per_sm = CTF_TC05_MINB;
            long long grid = (long long)sms * per_sm;
            const long long need = ((long long)k.nchunks + tc05::kWarpsT - 1) / tc05::kWarpsT;
            if (grid > need) grid = need;
            kern<<<(unsigned)(grid < 1 ? 1 : grid), tc05::kWarpsT * 32, dyn, stream>>>(k, mw);
            return cudaGetLastError();
        }
    }
    auto kern = use_fused<FMT>(k) ? lean_kernel_for<FMT, DBG, true>(k) : lean_kernel_for<FMT, DBG, false>(k);
    const size_t dyn = FMT == FMT_BC1 ? 0 : sizeof(TcWeights) + lean_warps<FMT>() * sizeof(TcScratch);
    int per_sm = 0;
    cudaError_t e;
    if (dyn > 0 && (e = mlp_smem_setup(kern, dyn, dev)) != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, lean_warps<FMT>() * 32, dyn);
    if (e != cudaSuccess) return e;
    const long long slots = (long long)sms * (per_sm > 0 ? per_sm : 1);
    long long ipw;
    if (FMT == FMT_BC1) {   // many short-lived CTAs; the block scheduler balances
        ipw = ((long long)k.nchunks + slots * lean_warps<FMT>() * CTF_BC1_ROUNDS / 2) / (slots * lean_warps<FMT>() * CTF_BC1_ROUNDS);
        ipw = ipw < 1 ? 1 : ipw > CTF_BC1_MAX_IPW ? CTF_BC1_MAX_IPW : ipw;
    } else {                // latent MLP: one CTA per slot (each CTA stages the MLP weights once)
        ipw = ((long long)k.nchunks + slots * lean_warps<FMT>() - 1) / (slots * lean_warps<FMT>());
        if (ipw < 1) ipw = 1;
    }
    k.ipc = (unsigned)(ipw * lean_warps<FMT>());
    long long grid = ((long long)k.nchunks + k.ipc - 1) / k.ipc;
    if (grid < 1) grid = 1;
#ifndef CTF_PDL_EARLY_DIV
#define CTF_PDL_EARLY_DIV 2  // early trigger when the grid fills at most 1/DIV of the resident CTA slots
#endif
    if (grid * CTF_PDL_EARLY_DIV <= slots) k.flags |= FLAG_PDL_EARLY;
    // launched as a programmatic dependent of the previous kernel on the stream (it waits for
    // it in-kernel, after its shared-memory prologue)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(lean_warps<FMT>() * 32);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, k, mw);
}

// the marked waves of k's frames: pass 0 lean fallback (BC1), pass 1 general; each pass at
// most one resident wave of CTAs
template <int FMT, bool DBG>
static cudaError_t launch_rest(const KArgs &k, const typename WeightsOf<FMT>::type &mw, int dev, int sms,
                               cudaStream_t stream) {
    const size_t dyn_mlp = FMT == FMT_BC1 ? 0 : sizeof(TcWeights) + kWarps * sizeof(TcScratch);
    const unsigned nrec = (unsigned)((long long)k.wpf * (k.nchunks / (unsigned)k.cpf));
    const long long groups = ((long long)nrec + 31) / 32;
    const int first = FMT == FMT_BC1 ? 0 : 1;
    cudaError_t e;
    // BC1 with CTF_REST_CONCURRENT: the third kernel (its waves routed by the lean kernel) first,
    // the wide-window kernel launched as its programmatic dependent right away (see the kernel)
    constexpr bool conc = FMT == FMT_BC1 && CTF_REST_CONCURRENT && !CTF_REST_MERGED;
    const int npass = CTF_REST_MERGED ? 1 : 2;
    for (int pi = first; pi < npass; ++pi) {
        const int pass = conc ? 1 - pi : pi;
        auto rest = ctf_collab_rest_kernel<DBG, false, FMT>;
        if constexpr (FMT == FMT_BC1)
            if (pass == 0) rest = ctf_collab_rest_kernel<DBG, true, FMT_BC1>;
        // BC1 third kernel: the 64 x 64 windows (CTF_REST_BIG) in dynamic shared memory
        const size_t dyn = FMT == FMT_BC1 ? (pass == 1 && CTF_REST_BIG ? kWarps * sizeof(WideSmemBig) : 0) : dyn_mlp;
        int per_sm = 0;
        if (dyn > 0 && (e = mlp_smem_setup(rest, dyn, dev)) != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rest, kWarps * 32, dyn);
        if (e != cudaSuccess) return e;
#ifndef CTF_THIRD_PER_SM
#define CTF_THIRD_PER_SM 3  // BC1 third kernel (runs alongside the wide-window kernel): CTAs per SM at most
#endif
        if (conc && pass == 1 && per_sm > CTF_THIRD_PER_SM) per_sm = CTF_THIRD_PER_SM;
        long long g2 = (long long)sms * (per_sm > 0 ? per_sm : 1);
        if (g2 * kWarps > groups) g2 = (groups + kWarps - 1) / kWarps;
        // programmatic dependent launch: this pass is launched while the previous kernel runs and
        // waits for it in-kernel (griddepcontrol.wait) — its launch latency overlaps the previous
        // pass instead of following it
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = dim3((unsigned)(g2 < 1 ? 1 : g2));
        cfg.blockDim = dim3(kWarps * 32);
        cfg.dynamicSmemBytes = dyn;
        cfg.stream = stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if ((e = cudaLaunchKernelEx(&cfg, rest, k, nrec, mw)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int FMT, bool DBG>
static cudaError_t launch_fast(KArgs k, const typename WeightsOf<FMT>::type &mw, cudaStream_t stream) {
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    if (FMT == FMT_BC1) {
        // as many runs per wave-row as fill every resident warp once (small calls are
        // latency-bound: a warp's waves are a dependent chain; equal-length runs keep the SMs
        // evenly loaded), between ceil(nwx / kChunk) (runs of <= kChunk waves, large batches)
        // and nwx / 2 (runs of >= 2 waves: pairs)
        const long long warps = (long long)sms * CTF_PAIR_MINB * kWarps;
        const unsigned frames = k.nrec / (unsigned)k.wpf;
        const long long rows = (long long)k.nwy * frames;
        const long long rmin = (k.nwx + kChunk - 1) / kChunk;
        const long long rmax = k.nwx / 2 > rmin ? k.nwx / 2 : rmin;
        long long R = warps / (rows > 0 ? rows : 1);
        R = R < rmin ? rmin : R > rmax ? rmax : R;
        k.cpr = (int)R;
        k.chunk = (int)((k.nwx + R - 1) / R);
        udiv_magic_host((unsigned)k.cpr, k.cpr_m, k.cpr_s);
        k.cpf = k.cpr * k.nwy;
        k.nchunks = (unsigned)((long long)k.cpf * frames);
    }
    if (use_fused<FMT>(k)) {   // one launch: the lean kernel finishes its own marked waves
        k.lists = nullptr;
        return launch_lean<FMT, DBG>(k, mw, dev, sms, stream);
    }
    if (k.lists) {   // work-list counters (the lists need no initialisation)
        k.lcnt = k.lists;
        k.lists += 64;
        if ((e = cudaMemsetAsync(k.lcnt, 0, 2 * sizeof(uint32_t), stream)) != cudaSuccess) return e;
    }
    if ((e = launch_lean<FMT, DBG>(k, mw, dev, sms, stream)) != cudaSuccess) return e;
    return launch_rest<FMT, DBG>(k, mw, dev, sms, stream);
}

template <int FMT, int MODE>
static cudaError_t launch_dbg(const KArgs &k, const typename WeightsOf<FMT>::type &mw, cudaStream_t stream) {
    // List and Mask 16x16 / 11x11 share the lean kernels: every lean exact window is <= 8x8,
    // inside both grids, so there Mask's success test is List's; the lean fallback kernel adds
    // the grid test for its wider windows.  Box has its own lean exact instantiation.
    if (CTF_FAST && MODE == MODE_COLLAB)
        return (k.flags & FLAG_DEBUG) ? launch_fast<FMT, true>(k, mw, stream) : launch_fast<FMT, false>(k, mw, stream);
    return (k.flags & FLAG_DEBUG) ? launch_one<FMT, MODE, true>(k, mw, stream)
                                  : launch_one<FMT, MODE, false>(k, mw, stream);
}

template <int FMT>
static cudaError_t launch_fmt(const KArgs &k, const typename WeightsOf<FMT>::type &mw, int mode, cudaStream_t stream) {
    switch (mode) {
    case MODE_4TAP: return launch_dbg<FMT, MODE_4TAP>(k, mw, stream);
    case MODE_STF: return launch_dbg<FMT, MODE_STF>(k, mw, stream);
    case MODE_WC: return launch_dbg<FMT, MODE_WC>(k, mw, stream);
    default: return launch_dbg<FMT, MODE_COLLAB>(k, mw, stream);
    }
}

#ifndef CTF_TU_FMT
#error "compile ctf_filter.cu with -DCTF_TU_FMT=1 (BC1) or =2 (latent MLP)"
#endif
#if CTF_TU_FMT == 1
int launches_per_pass(int fmt, int mode, int filter, long long waves, unsigned flags) {
    if (!CTF_FAST || mode < MODE_COLLAB || mode > MODE_COLLAB + 3 || filter != 0)
        return 1;   // List (3), Box (4), Mask16 (5), Mask11 (6) run the lean kernels
    if (fmt == FMT_BC1 && waves <= CTF_FUSED_MAX_WAVES && !(flags & FLAG_SEPARATE_PASSES)) return 1;   // fused
    return fmt == FMT_BC1 ? (CTF_REST_MERGED ? 2 : 3) : 2;   // latent MLP: lean exact + general
}

cudaError_t launch_filter_bc1(const LaunchArgs &a, cudaStream_t stream) {
#else
cudaError_t launch_filter_mlp(const LaunchArgs &a, cudaStream_t stream) {
#endif
    KArgs k;
    k.tex.W = a.W;
    k.tex.H = a.H;
    k.tex.bc1 = reinterpret_cast<const uint2 *>(a.tex_data);
    k.tex.latent = reinterpret_cast<const uint4 *>(a.tex_data);
    k.tex.mlp_dev = a.mlp;
    k.uv = reinterpret_cast<const float2 *>(a.uv);
    k.grad = reinterpret_cast<const uint2 *>(a.grad);
    k.out = reinterpret_cast<float4 *>(a.out);
    k.rec = a.rec;
    k.dbg_pid = a.dbg_pid;
    k.dbg_sel = a.dbg_sel;
    k.dbg_unread = a.dbg_unread;
    k.lists = a.lists;
    k.lcnt = nullptr;
    k.Wf = a.Wf;
    k.Hf = a.Hf;
    k.nwx = (a.Wf + 7) / 8;
    k.nwy = (a.Hf + 3) / 4;
    k.wpf = k.nwx * k.nwy;
    k.fpx = (unsigned)a.Wf * (unsigned)a.Hf;
    k.chunk = kChunk;
    k.cpr = (k.nwx + kChunk - 1) / kChunk;
    k.cpf = k.cpr * k.nwy;
    k.nchunks = (unsigned)((long long)k.cpf * a.frames);
    k.nrec = (unsigned)((long long)k.wpf * a.frames);
    udiv_magic_host((unsigned)k.wpf, k.wpf_m, k.wpf_s);
    udiv_magic_host((unsigned)k.nwx, k.nwx_m, k.nwx_s);
    udiv_magic_host((unsigned)k.cpr, k.cpr_m, k.cpr_s);
    k.Wflt = (float)a.W;
    k.Hflt = (float)a.H;
    k.Wm1 = a.W - 1;
    k.Hm1 = a.H - 1;
    k.fallback = a.fallback;
    k.variant = a.mode >= 4 ? a.mode - 3 : VAR_LIST;   // BOX / MASK16 / MASK11 run in the COLLAB kernel
    k.flags = a.flags;
    k.frame_index = a.frame_index;
    k.row0 = a.row0;
    k.seed_lo = (uint32_t)a.seed;
    k.seed_hi = (uint32_t)(a.seed >> 32);
    for (int r = 0; r < 10; ++r) {   // the key schedule of philox4x32_10, precomputed
        k.rk[0][r] = k.seed_lo + (uint32_t)r * 0x9E3779B9u;
        k.rk[1][r] = k.seed_hi + (uint32_t)r * 0xBB67AE85u;
    }
#if CTF_TU_FMT == 1
    return launch_fmt<FMT_BC1>(k, NoWeights{}, a.mode, stream);
#else
    static_assert(sizeof(MlpWeights) == sizeof(float) * kMlpParams, "weight layout");
    MlpWeights mw;
    const cudaError_t e = mlp_weights_by_value(a, stream, mw.v);
    if (e != cudaSuccess) return e;
    return launch_fmt<FMT_MLP>(k, mw, a.mode, stream);
#endif
}

}  // namespace ctf
