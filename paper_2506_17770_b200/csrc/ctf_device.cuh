// ctf_device.cuh — device building blocks of the CTF hot path (sm_100a).
//
// Independent of the CPU oracle: nothing here is shared with oracle/.
// P:n = PAPER.md line; R-n = DESIGN.md reading.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace ctf {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t INVALID_ID = 0xffffffffu;

enum { FMT_BC1 = 1, FMT_MLP = 2 };
enum { MODE_4TAP = 0, MODE_STF = 1, MODE_WC = 2, MODE_COLLAB = 3 };
enum { FB_STF = 0, FB_WC = 1, FB_C = 2, FB_CPLUS = 3 };
enum { FLAG_DEBUG = 1u, FLAG_FORCE_FALLBACK = 2u, FLAG_SEPARATE_PASSES = 4u };
// internal (set by the launcher, never by callers): the lean kernel's grid is one wave of
// resident CTAs, so it lets the next kernel on the stream launch at once (PDL)
enum : uint32_t { FLAG_PDL_EARLY = 1u << 30 };
enum { PATH_EXACT = 0, PATH_FB_STF = 1, PATH_FB_WC = 2, PATH_FB_C = 3, PATH_FB_CPLUS = 4,
       PATH_4TAP = 5, PATH_STF = 6, PATH_WC = 7 };

#ifndef CTF_LANEID_SREG
#define CTF_LANEID_SREG 1
#endif
// the lane index: %laneid is one S2R when ptxas rematerialises it (threadIdx.x & 31 is two)
__device__ __forceinline__ unsigned lane_id() {
#if CTF_LANEID_SREG
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
#else
    return threadIdx.x & 31u;
#endif
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------- streaming I/O
__device__ __forceinline__ float2 ld_stream_f2(const float2 *p) {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];"
                 : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream_u2(const uint2 *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
// predicated streaming loads: the destination keeps its prior value when pred == 0
__device__ __forceinline__ void ld_stream_f2_if(float2 &r, const float2 *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];\n\t}"
                 : "+f"(r.x), "+f"(r.y) : "l"(p), "r"((unsigned)pred));
}
__device__ __forceinline__ void ld_stream_u2_if(uint2 &r, const uint2 *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];\n\t}"
                 : "+r"(r.x), "+r"(r.y) : "l"(p), "r"((unsigned)pred));
}
__device__ __forceinline__ void ld_u32_if(uint32_t &r, const uint32_t *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.cg.u32 %0, [%1];\n\t}"
                 : "+r"(r) : "l"(p), "r"((unsigned)pred));
}
// predicated global atomic add / store without a branch (a divergent branch anywhere in a
// loop makes ptxas guard the loop's warp collectives with divergence checks)
__device__ __forceinline__ uint32_t atom_add_if(uint32_t *p, uint32_t v, bool pred) {
    uint32_t old = 0u;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.global.add.u32 %0, [%1], %2;\n\t}"
                 : "+r"(old) : "l"(p), "r"(v), "r"((unsigned)pred) : "memory");
    return old;
}
__device__ __forceinline__ void st_u32_if(uint32_t *p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}"
                 ::"l"(p), "r"(v), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ void st_stream_f4(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// shared-memory load from a 32-bit shared address
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
// predicated shared store without a branch (keeps the warp provably converged)
__device__ __forceinline__ void st_shared_u32_if(uint32_t *p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                 ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ void st_shared_f4_if(float4 *p, float4 v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n\t}"
                 ::"r"((unsigned)__cvta_generic_to_shared(p)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((unsigned)pred)
                 : "memory");
}
__device__ __forceinline__ void st_shared_u8_if(uint8_t *p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u8 [%0], %1;\n\t}"
                 ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v), "r"((unsigned)pred) : "memory");
}

// ---------------------------------------------------------- Philox4x32-10 (R-11)
// Salmon et al. SC'11; counter (x, y, frame, 0), key (seed_lo, seed_hi).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}
// The same with the round keys precomputed (k0[r] = k0 + r * 0x9E3779B9, k1[r] likewise):
// kernel-parameter arrays, so each key is a constant-bank operand of the XOR.
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t (&k0)[10], const uint32_t (&k1)[10]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0[r], lo1, hi0 ^ c.w ^ k1[r], lo0);
    }
    return c;
}
// uniform in [0,1) on the 2^-24 grid: exact in fp32 (R-11)
__device__ __forceinline__ float unit24(uint32_t r) { return __uint2float_rn(r >> 8) * 5.9604644775390625e-08f; }

// ------------------------------------------------------- packed fp32 (sm_100 FFMA2)
// Two fp32 lanes in one 64-bit register pair; each lane is an ordinary IEEE fp32
// operation with one rounding, so results equal the scalar instructions bit for bit.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 f2unpack(uint64_t r) {
    float2 v;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// (2^23 + v) bit patterns of the four channels -> v / 255 as v * fl(1/255) (R-9): FADD2
// removes the 2^23 (exact), one FMUL2 scales.  Within 1 ulp (6e-8) of the correctly rounded
// quotient for every v in [0, 255] (exact for 130 of the 256 values; checked exhaustively,
// DESIGN.md R-9) — every BC1 path converts through here, so exact waves stay bit-identical to
// 4-tap.  No I2F, no correction step.
__device__ __forceinline__ float4 magic_unorm(uint32_t r, uint32_t g, uint32_t b, uint32_t a) {
    uint64_t rg = f2pack(__uint_as_float(r), __uint_as_float(g));
    uint64_t ba = f2pack(__uint_as_float(b), __uint_as_float(a));
    const uint64_t mag = f2pack(-8388608.0f, -8388608.0f), rc = f2pack(1.0f / 255.0f, 1.0f / 255.0f);
    const float2 x = f2unpack(fmul2(fadd2(rg, mag), rc)), y = f2unpack(fmul2(fadd2(ba, mag), rc));
    return make_float4(x.x, x.y, y.x, y.y);
}
// RGBA8 -> v / 255 per channel: a byte permute places each byte under the 2^23 exponent.
__device__ __forceinline__ float4 rgba8_unorm(uint32_t v) {
    return magic_unorm(__byte_perm(v, 0x4B000000u, 0x7540), __byte_perm(v, 0x4B000000u, 0x7541),
                       __byte_perm(v, 0x4B000000u, 0x7542), __byte_perm(v, 0x4B000000u, 0x7543));
}

// Exact bilinear blend (c8 / R-8): per channel c = fma(w3,p3, fma(w2,p2, fma(w1,p1, w0*p0))),
// two channels per FFMA2.  Every exact path (COLLAB fast / generic, 4TAP, Eq. 1's
// all-known case) calls this, so they agree bit for bit.
__device__ __forceinline__ float4 blend4f(const float4 (&p)[4], const float (&w)[4]) {
    uint64_t rg = fmul2(f2pack(p[0].x, p[0].y), f2pack(w[0], w[0]));
    uint64_t ba = fmul2(f2pack(p[0].z, p[0].w), f2pack(w[0], w[0]));
#pragma unroll
    for (int k = 1; k < 4; ++k) {
        rg = ffma2(f2pack(p[k].x, p[k].y), f2pack(w[k], w[k]), rg);
        ba = ffma2(f2pack(p[k].z, p[k].w), f2pack(w[k], w[k]), ba);
    }
    const float2 a = f2unpack(rg), b = f2unpack(ba);
    return make_float4(a.x, a.y, b.x, b.y);
}

// ------------------------------------------------------------------ texels
// A produced texel and how lanes exchange it (step 3 "gather"; WaveReadLaneAt).
template <int FMT> struct Texel;

template <> struct Texel<FMT_BC1> {
    uint32_t v;  // RGBA8 packed: one 32-bit shuffle per texel
    __device__ __forceinline__ static Texel shfl(Texel t, int src) { return {__shfl_sync(FULL, t.v, src)}; }
    __device__ __forceinline__ float ch(int c) const { return (float)((v >> (8 * c)) & 255u); }
    __device__ __forceinline__ void expand(float (&c)[4]) const;         // exact v in [0, 255]
    __device__ __forceinline__ void expand_biased(float (&c)[4]) const;  // 1024 + v (no constant operand)
    __device__ __forceinline__ float4 to_f4() const { return rgba8_unorm(v); }  // v / 255 (R-9)
    __device__ __forceinline__ static Texel zero() { return {0u}; }
    static constexpr float kScale = 1.0f / 255.0f;  // bytes -> [0,1] (R-9)
    static constexpr float kBias = 1024.0f;
};

template <> struct Texel<FMT_MLP> {
    float4 v;
    __device__ __forceinline__ static Texel shfl(Texel t, int src) {
        return {make_float4(__shfl_sync(FULL, t.v.x, src), __shfl_sync(FULL, t.v.y, src),
                            __shfl_sync(FULL, t.v.z, src), __shfl_sync(FULL, t.v.w, src))};
    }
    __device__ __forceinline__ float ch(int c) const { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }
    __device__ __forceinline__ void expand(float (&c)[4]) const { c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w; }
    __device__ __forceinline__ void expand_biased(float (&c)[4]) const { expand(c); }
    __device__ __forceinline__ float4 to_f4() const { return v; }
    __device__ __forceinline__ static Texel zero() { return {make_float4(0.f, 0.f, 0.f, 0.f)}; }
    static constexpr float kScale = 1.0f;
    static constexpr float kBias = 0.0f;
};

struct TexArgs {
    int W, H;
    const uint2 *bc1;       // BC1 blocks
    const uint4 *latent;    // 8 x fp16 per latent texel
    const float *mlp_dev;   // MLP weights in the ABI layout (per-lane rows of the batched decoder)
};

constexpr int kMlpWeights = 32 * 12 + 32 + 32 * 32 + 32 + 4 * 32 + 4;  // 1604 (R-10)
// Latent-MLP weights travel BY VALUE in the kernel parameter block (constant bank 0):
// every lane reads the same weight at the same time, so FFMA takes it straight from
// the constant cache with no load instruction.  BC1 kernels get an empty struct.
struct alignas(16) MlpWeights {   // 16-B aligned in the kernel parameter block (vector constant loads)
    float v[kMlpWeights];
};
struct NoWeights {};
template <int FMT> struct WeightsOf { using type = NoWeights; };
template <> struct WeightsOf<2> { using type = MlpWeights; };

// Synthetic BC1-style decode of texel (x, y) (R-9).  Integer only and branch-free.
// Both endpoints are expanded at once in 16-bit lanes (e0 low, e1 high); the palette
// entry wa*e0 + wb*e1 is one IMAD against M = (wa << 16) | wb (bits 16-31 of the
// product), then /1, /2 or /3 as (v * {2048, 1024, 683}) >> 11 — exact for v <= 765
// (checked exhaustively, R-9).
// Channel products before the final >> 11 (palette value = product >> 11) and alpha.
struct Bc1Raw {
    uint32_t r, g, b;
    bool opaque;
};
__device__ __forceinline__ Bc1Raw bc1_raw(const TexArgs &t, int x, int y) {
    const uint2 b = __ldg(t.bc1 + ((unsigned)(y >> 2) * (unsigned)(t.W >> 2) + (unsigned)(x >> 2)));
    const uint32_t shift = 2u * ((((unsigned)y & 3u) << 2) | ((unsigned)x & 3u));
    const uint32_t code = (b.y >> shift) & 3u;
    const bool four = (b.x & 0xffffu) > (b.x >> 16);
    uint32_t rp = (b.x >> 11) & 0x001F001Fu;
    rp = ((rp << 3) | (rp >> 2)) & 0x00FF00FFu;
    uint32_t gp = (b.x >> 5) & 0x003F003Fu;
    gp = ((gp << 2) | (gp >> 4)) & 0x00FF00FFu;
    uint32_t bp = b.x & 0x001F001Fu;
    bp = ((bp << 3) | (bp >> 2)) & 0x00FF00FFu;
    const uint32_t i = code | (four ? 4u : 0u);
    const uint32_t nib = (0x96410541u >> (4u * i)) & 15u;
    const uint32_t M = ((nib & 3u) << 16) | (nib >> 2);
    const uint32_t mul = code < 2u ? 2048u : (four ? 683u : 1024u);
    return {((rp * M) >> 16) * mul, ((gp * M) >> 16) * mul, ((bp * M) >> 16) * mul, four || code != 3u};
}
// Texel (x, y) straight to v / 255 per channel (= rgba8_unorm(bc1_decode(...)) bit for bit):
// the palette bytes land under the 2^23 exponent with one LEA.HI each, no RGBA8 packing.
__device__ __forceinline__ float4 bc1_decode_unorm(const TexArgs &t, int x, int y) {
    const Bc1Raw q = bc1_raw(t, x, y);
    return magic_unorm((q.r >> 11) + 0x4B000000u, (q.g >> 11) + 0x4B000000u, (q.b >> 11) + 0x4B000000u,
                       q.opaque ? 0x4B0000FFu : 0x4B000000u);
}

// The same with the per-index constants from a shared-memory table (one LDS.128 instead of
// ~10 instructions of table-in-register arithmetic): entry i = code | four << 2 holds
// {M, mul, alpha bits under 2^23, 0}; fill it with bc1_lut_entry(i).
__device__ __forceinline__ uint4 bc1_lut_entry(uint32_t i) {
    const uint32_t code = i & 3u;
    const bool four = i >= 4u;
    const uint32_t nib = (0x96410541u >> (4u * i)) & 15u;
    return make_uint4(((nib & 3u) << 16) | (nib >> 2), code < 2u ? 2048u : (four ? 683u : 1024u),
                      (four || code != 3u) ? 0x4B0000FFu : 0x4B000000u, 0u);
}
// BC1 block of texel (x, y) (the load of bc1_decode_unorm_lut, issued ahead by the paired path)
__device__ __forceinline__ uint2 bc1_block(const TexArgs &t, int x, int y) {
    return __ldg(t.bc1 + ((unsigned)(y >> 2) * (unsigned)(t.W >> 2) + (unsigned)(x >> 2)));
}
__device__ __forceinline__ float4 bc1_unorm_from_block(uint2 b, int x, int y, const uint4 *lut);
__device__ __forceinline__ float4 bc1_decode_unorm_lut(const TexArgs &t, int x, int y, const uint4 *lut) {
    return bc1_unorm_from_block(bc1_block(t, x, y), x, y, lut);
}
__device__ __forceinline__ float4 bc1_unorm_from_block(uint2 b, int x, int y, const uint4 *lut) {
    const uint32_t shift = 2u * ((((unsigned)y & 3u) << 2) | ((unsigned)x & 3u));
    const uint32_t code = (b.y >> shift) & 3u;
    const bool four = (b.x & 0xffffu) > (b.x >> 16);
    const uint4 e = lut[code | (four ? 4u : 0u)];
    uint32_t rp = (b.x >> 11) & 0x001F001Fu;
    rp = ((rp << 3) | (rp >> 2)) & 0x00FF00FFu;
    uint32_t gp = (b.x >> 5) & 0x003F003Fu;
    gp = ((gp << 2) | (gp >> 4)) & 0x00FF00FFu;
    uint32_t bp = b.x & 0x001F001Fu;
    bp = ((bp << 3) | (bp >> 2)) & 0x00FF00FFu;
    return magic_unorm((((rp * e.x) >> 16) * e.y >> 11) + 0x4B000000u, (((gp * e.x) >> 16) * e.y >> 11) + 0x4B000000u,
                       (((bp * e.x) >> 16) * e.y >> 11) + 0x4B000000u, e.z);
}

__device__ __forceinline__ uint32_t bc1_decode(const TexArgs &t, int x, int y) {
    const uint2 b = __ldg(t.bc1 + ((unsigned)(y >> 2) * (unsigned)(t.W >> 2) + (unsigned)(x >> 2)));
    const uint32_t shift = 2u * ((((unsigned)y & 3u) << 2) | ((unsigned)x & 3u));
    const uint32_t code = (b.y >> shift) & 3u;
    const bool four = (b.x & 0xffffu) > (b.x >> 16);
    uint32_t rp = (b.x >> 11) & 0x001F001Fu;
    rp = ((rp << 3) | (rp >> 2)) & 0x00FF00FFu;
    uint32_t gp = (b.x >> 5) & 0x003F003Fu;
    gp = ((gp << 2) | (gp >> 4)) & 0x00FF00FFu;
    uint32_t bp = b.x & 0x001F001Fu;
    bp = ((bp << 3) | (bp >> 2)) & 0x00FF00FFu;
    // (wa, wb) for index code | four << 2, 4 bits each: wa in bits 0-1, wb in bits 2-3
    //   4-colour: {c0, c1, (2c0+c1)/3, (c0+2c1)/3}; 3-colour: {c0, c1, (c0+c1)/2, 0}
    const uint32_t i = code | (four ? 4u : 0u);
    const uint32_t nib = (0x96410541u >> (4u * i)) & 15u;
    const uint32_t M = ((nib & 3u) << 16) | (nib >> 2);
    const uint32_t mul = code < 2u ? 2048u : (four ? 683u : 1024u);
    const uint32_t r = (((rp * M) >> 16) * mul) >> 11;
    const uint32_t g = (((gp * M) >> 16) * mul) >> 11;
    const uint32_t bb = (((bp * M) >> 16) * mul) >> 11;
    const uint32_t a = (four || code != 3u) ? 0xff000000u : 0u;
    return r | (g << 8) | (bb << 16) | a;
}

// fp16 -> fp32 convert-and-add in one instruction (PTX 8.6 mixed precision, sm_100+).
__device__ __forceinline__ float f16_add_f32(unsigned short h, float c) {
    float d;
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"(h), "f"(c));
    return d;
}
// fp32 = fp16 * fp16 + fp32 with one rounding (PTX 8.6 mixed precision, sm_100+).
__device__ __forceinline__ float fma_f32_f16(unsigned short a, unsigned short b, float c) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
    return d;
}
// RGBA8 -> 4 exact floats in [0,255]: two byte permutes build half2 (1024 + v) pairs
// (0x64xx), then each half is converted while subtracting 1024 (no slow I2F).
__device__ __forceinline__ void rgba8_to_float(uint32_t v, float (&c)[4]) {
    const uint32_t rg = __byte_perm(v, 0x64646464u, 0x4140);
    const uint32_t ba = __byte_perm(v, 0x64646464u, 0x4342);
    c[0] = f16_add_f32((unsigned short)(rg & 0xffffu), -1024.0f);
    c[1] = f16_add_f32((unsigned short)(rg >> 16), -1024.0f);
    c[2] = f16_add_f32((unsigned short)(ba & 0xffffu), -1024.0f);
    c[3] = f16_add_f32((unsigned short)(ba >> 16), -1024.0f);
}

// Latent + MLP decode (R-10; NTC-style inference-on-sample).  fp32 FFMA.
// Weights are read from the kernel parameter block with compile-time offsets.
// The 12 MLP inputs of texel (x, y): bilinear latent sample + 4 positional features.
__device__ __forceinline__ void mlp_features(const TexArgs &t, int x, int y, float (&in)[12]) {
    const int lw = t.W >> 2, lh = t.H >> 2;
    // sample point ((x-1.5)/4, (y-1.5)/4): integer part and phase in eighths (exact weights)
    const int gx8 = 2 * x - 3, gy8 = 2 * y - 3;                 // 8 * position
    const int ix = gx8 >> 3, iy = gy8 >> 3;                      // floor
    const float fx = (float)(gx8 & 7) * 0.125f, fy = (float)(gy8 & 7) * 0.125f;
    const int x0 = min(max(ix, 0), lw - 1), x1 = min(max(ix + 1, 0), lw - 1);
    const int y0 = min(max(iy, 0), lh - 1), y1 = min(max(iy + 1, 0), lh - 1);
    const uint4 q00 = __ldg(t.latent + (size_t)y0 * lw + x0), q01 = __ldg(t.latent + (size_t)y0 * lw + x1);
    const uint4 q10 = __ldg(t.latent + (size_t)y1 * lw + x0), q11 = __ldg(t.latent + (size_t)y1 * lw + x1);
    const float w00 = (1.f - fx) * (1.f - fy), w01 = fx * (1.f - fy), w10 = (1.f - fx) * fy, w11 = fx * fy;
    const uint32_t *a0 = &q00.x, *a1 = &q01.x, *a2 = &q10.x, *a3 = &q11.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 v0 = __half22float2(*reinterpret_cast<const __half2 *>(a0 + k));
        const float2 v1 = __half22float2(*reinterpret_cast<const __half2 *>(a1 + k));
        const float2 v2 = __half22float2(*reinterpret_cast<const __half2 *>(a2 + k));
        const float2 v3 = __half22float2(*reinterpret_cast<const __half2 *>(a3 + k));
        in[2 * k] = fmaf(w11, v3.x, fmaf(w10, v2.x, fmaf(w01, v1.x, w00 * v0.x)));
        in[2 * k + 1] = fmaf(w11, v3.y, fmaf(w10, v2.y, fmaf(w01, v1.y, w00 * v0.y)));
    }
    in[8] = (float)((x & 3) * 2 - 3) * 0.25f;
    in[9] = (float)((y & 3) * 2 - 3) * 0.25f;
    in[10] = ((x >> 2) & 1) ? 0.5f : -0.5f;
    in[11] = ((y >> 2) & 1) ? 0.5f : -0.5f;
}

// Latent + MLP decode of one texel by one lane (R-10; NTC-style inference-on-sample,
// P:729-752).  fp32 FFMA; weights read from the kernel parameter block with
// compile-time offsets.  The wave-batched decoder in ctf_filter.cu performs the same
// operations in the same order per output, so both give bit-identical texels.
__device__ __forceinline__ float4 mlp_decode(const TexArgs &t, const MlpWeights &wt, int x, int y) {
    const float *w = wt.v;
    float in[12];
    mlp_features(t, x, y, in);
    // Kernel weight layout (repacked by the launcher so every access is contiguous and
    // the compiler can fetch 4 weights per LDCU.128): W1[k][12], b1[32], W2T[k][j] =
    // W2[j][k], b2[32], W3T[j][4] = W3[c][j], b3[4].
    const float *W1 = w, *b1 = W1 + 32 * 12, *W2T = b1 + 32, *b2 = W2T + 32 * 32, *W3T = b2 + 32, *b3 = W3T + 4 * 32;
    // Outer-product order keeps ~50 values live instead of ~100: each hidden unit k of
    // layer 1 is formed and immediately scattered into the 32 layer-2 accumulators;
    // then each layer-2 unit feeds the 4 outputs.  Same 1536 FMAs.
    float acc2[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc2[j] = b2[j];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        float h = b1[k];
#pragma unroll
        for (int i = 0; i < 12; ++i) h = fmaf(W1[k * 12 + i], in[i], h);
        h = fmaxf(h, 0.f);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc2[j] = fmaf(W2T[k * 32 + j], h, acc2[j]);
    }
    float o[4] = {b3[0], b3[1], b3[2], b3[3]};
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const float h = fmaxf(acc2[j], 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = fmaf(W3T[j * 4 + c], h, o[c]);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] = fminf(fmaxf(o[c], 0.f), 1.f);
    return make_float4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ void Texel<FMT_BC1>::expand(float (&c)[4]) const { rgba8_to_float(v, c); }
__device__ __forceinline__ void Texel<FMT_BC1>::expand_biased(float (&c)[4]) const {
    const uint32_t rg = __byte_perm(v, 0x64646464u, 0x4140);
    const uint32_t ba = __byte_perm(v, 0x64646464u, 0x4342);
    c[0] = f16_add_f32((unsigned short)(rg & 0xffffu), 0.0f);
    c[1] = f16_add_f32((unsigned short)(rg >> 16), 0.0f);
    c[2] = f16_add_f32((unsigned short)(ba & 0xffffu), 0.0f);
    c[3] = f16_add_f32((unsigned short)(ba >> 16), 0.0f);
}

__device__ __forceinline__ Texel<FMT_BC1> produce(const TexArgs &t, const NoWeights &, uint32_t x, uint32_t y) {
    return {bc1_decode(t, (int)x, (int)y)};
}
__device__ __forceinline__ Texel<FMT_MLP> produce(const TexArgs &t, const MlpWeights &w, uint32_t x, uint32_t y) {
    return {mlp_decode(t, w, (int)x, (int)y)};
}

// ------------------------------------------------------------- warp sorting
// Bitonic sort of one 32-bit key per lane, ascending by lane (shfl_xor network).
__device__ __forceinline__ uint32_t warp_sort32(uint32_t key) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint32_t other = __shfl_xor_sync(FULL, key, j);
            const bool asc = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            key = (lower == asc) ? min(key, other) : max(key, other);
        }
    }
    return key;
}

// Bitonic sort of 128 keys held 4 per lane (element e = 4*lane + r), ascending in e.
__device__ __forceinline__ void warp_sort128(uint32_t (&k)[4]) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 128; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            if (j >= 4) {
                const int lj = j >> 2;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t other = __shfl_xor_sync(FULL, k[r], lj);
                    const unsigned e = 4u * lane + r;
                    const bool asc = (e & size) == 0;
                    const bool lower = (lane & lj) == 0;
                    k[r] = (lower == asc) ? min(k[r], other) : max(k[r], other);
                }
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r & j) continue;
                    const unsigned e = 4u * lane + r;
                    const bool asc = (e & size) == 0;
                    const uint32_t a = k[r], b = k[r | j];
                    k[r] = asc ? min(a, b) : max(a, b);
                    k[r | j] = asc ? max(a, b) : min(a, b);
                }
            }
        }
    }
}

// lower_bound of `q` in a sorted shared array of 32 keys; returns index in [0, 32].
__device__ __forceinline__ int lower_bound32(const uint32_t *s, uint32_t q) {
    int pos = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
        if (s[pos + step - 1] < q) pos += step;
    return (pos < 31 || s[31] >= q) ? pos : 32;
}

}  // namespace ctf
