// ctf_filter.cu — the collaborative texture filtering kernel (sm_100a).
//
// One 8x4-pixel wave = one warp.  Persistent grid: each warp walks
// waves w = gwarp, gwarp + nwarps, ... over all frames of the batch.  Per wave:
//   a1 load uv/grad (coalesced 64-B row segments), active mask A = ballot
//   a2 footprint: fx = u*W - 0.5, floor, clamp, 4 texel ids
//   a3 collect: exact unique set U of the wave's footprint texels (List
//      semantics) in canonical ascending-id order (Mask h-order,
//      P:389-399).  Fast path: AABB by 4 redux.sync, then a row-major bitmask
//      of the AABB with power-of-two pitch (<= 128 bits) OR-reduced by
//      redux.sync (the WaveActiveBitOr of P:377) and popc ranks
//      (h^-1).  Slow path: bitonic sort of the 128 footprint keys.
//   a4 decide: exact iff n <= popc(A)
//   a5 produce: active rank r < n produces texel U[r] (lane h(r,A))
//   a6 gather + blend: 4 __shfl_sync (WaveReadLaneAt) + fma chain
//   a7 fallback (n > a): STF / WC stand-in / C (Eq. 1) / C+ (Eq. 2)
//   a8 per-wave record
#include <climits>
#include <cmath>

#include "ctf_device.cuh"
#include "ctf_internal.h"

namespace ctf {

constexpr int kWarps = 8;  // warps per CTA

struct KArgs {
    TexArgs tex;
    const float2 *uv;
    const uint2 *grad;
    float4 *out;
    uint32_t *rec;
    uint32_t *dbg_pid, *dbg_sel, *dbg_unread;
    long long total_waves;
    int Wf, Hf, nwx, wpf;  // waves per frame
    float Wflt, Hflt;
    int fallback;
    uint32_t flags, frame_index, seed_lo, seed_hi;
};

struct WarpSmem {
    uint32_t tbl[32];       // rank -> texel (exact path) / sorted planned ids P (C+)
    uint32_t sorted[32];    // sorted (id << 5 | lane) of produced texels (fallback gather)
    uint8_t lane_of_rank[32];
    uint8_t rank_of[128];   // slow-path collect: (lane*4 + corner) -> rank
};

// Per-lane footprint of one pixel (a2).
struct Foot {
    int xa, xb, ya, yb;     // clamped texel columns / rows
    uint32_t id[4];         // UL, UR, LL, LR
    float s, t;             // fp32 fractional position (decides coordinates)
    float w[4];             // fp32 weights, each product rounded once (R-3)
};

__device__ __forceinline__ void make_weights(Foot &f) {
    const float oms = __fsub_rn(1.0f, f.s), omt = __fsub_rn(1.0f, f.t);
    f.w[0] = __fmul_rn(oms, omt);
    f.w[1] = __fmul_rn(f.s, omt);
    f.w[2] = __fmul_rn(oms, f.t);
    f.w[3] = __fmul_rn(f.s, f.t);
}

__device__ __forceinline__ void make_ids(Foot &f, int W) {
    f.id[0] = (uint32_t)(f.ya * W + f.xa);
    f.id[1] = (uint32_t)(f.ya * W + f.xb);
    f.id[2] = (uint32_t)(f.yb * W + f.xa);
    f.id[3] = (uint32_t)(f.yb * W + f.xb);
}

__device__ __forceinline__ Foot footprint(float2 uv, const KArgs &a) {
    Foot f;
    // R-2: clamp to [-16, 16] (NaN v -> -16), two fp32 roundings, floor, exact s
    const float uc = fminf(fmaxf(uv.x, -16.0f), 16.0f), vc = fminf(fmaxf(uv.y, -16.0f), 16.0f);
    const float fx = __fsub_rn(__fmul_rn(uc, a.Wflt), 0.5f), fy = __fsub_rn(__fmul_rn(vc, a.Hflt), 0.5f);
    const float flx = floorf(fx), fly = floorf(fy);
    const int x0 = (int)flx, y0 = (int)fly;
    f.s = __fsub_rn(fx, flx);
    f.t = __fsub_rn(fy, fly);
    const int W = a.tex.W, H = a.tex.H;
    f.xa = min(max(x0, 0), W - 1);
    f.xb = min(max(x0 + 1, 0), W - 1);
    f.ya = min(max(y0, 0), H - 1);
    f.yb = min(max(y0 + 1, 0), H - 1);
    make_ids(f, W);
    make_weights(f);
    return f;
}

__device__ __forceinline__ int corner_x(const Foot &f, int k) { return (k & 1) ? f.xb : f.xa; }
// runtime-indexed corner id without local-memory indexing
__device__ __forceinline__ uint32_t corner_id(const Foot &f, int k) {
    return k == 0 ? f.id[0] : k == 1 ? f.id[1] : k == 2 ? f.id[2] : f.id[3];
}
__device__ __forceinline__ int corner_y(const Foot &f, int k) { return (k & 2) ? f.yb : f.ya; }

// Exact bilinear of 4 gathered texels (c8): same code in 4TAP and COLLAB-exact,
// so the two are bit-identical on exact waves.
template <int FMT>
__device__ __forceinline__ float4 blend4(const Texel<FMT> (&p)[4], const float (&w)[4]) {
    float c[4];
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
        c[ch] = fmaf(w[3], p[3].ch(ch), fmaf(w[2], p[2].ch(ch), fmaf(w[1], p[1].ch(ch), w[0] * p[0].ch(ch))));
    const float sc = Texel<FMT>::kScale;
    return make_float4(c[0] * sc, c[1] * sc, c[2] * sc, c[3] * sc);
}

template <int FMT>
__device__ __forceinline__ float4 scaled(const Texel<FMT> &p) {
    const float sc = Texel<FMT>::kScale;
    return make_float4(p.ch(0) * sc, p.ch(1) * sc, p.ch(2) * sc, p.ch(3) * sc);
}

// Eq. 2 generalised to a active lanes (R-18 iv), round half up.
__device__ __forceinline__ int eq2_lane_rank(int j, int np, int na) {
    if (np >= na - 1) return 0;
    const int num = 2 * (na - 1) * (j - np) + (na - 1 - np);
    const int den = 2 * (na - 1 - np);
    return num / den;
}

// STF corner (R-12): dx = (u0 < s), dy = (u1 < t).
__device__ __forceinline__ int stf_corner(const Foot &f, uint4 r) {
    return (unit24(r.x) < f.s ? 1 : 0) + (unit24(r.y) < f.t ? 2 : 0);
}

// Fallback gather + combine (c14-c16, c19).  Every lane holds its produced texel
// (`val`, id `prod` or INVALID).  Each lane looks up its distinct nonzero-weight
// footprint texels among the produced ones (sorted keys + binary search in smem),
// shuffles the values in and applies Eq. 1 (wc = false) or the WC stand-in.
template <int FMT>
__device__ __forceinline__ float4 fallback_gather(const Foot &f, bool active, uint32_t prod, const Texel<FMT> &val,
                                                  bool wc, WarpSmem &s) {
    const unsigned lane = lane_id();
    const uint32_t key = (active && prod != INVALID_ID) ? ((prod << 5) | lane) : INVALID_ID;
    s.sorted[lane] = warp_sort32(key);
    __syncwarp();
    // distinct corners in first-occurrence order with merged fp32 weights
    bool first[4];
    float dw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        first[k] = true;
        dw[k] = f.w[k];
    }
#pragma unroll
    for (int k = 1; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < k; ++j)
            if (first[j] && first[k] && f.id[j] == f.id[k]) {
                first[k] = false;
                dw[j] = __fadd_rn(dw[j], f.w[k]);
            }
    int src[4];
    bool known[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        known[k] = false;
        src[k] = (int)lane;
        if (active && first[k] && dw[k] != 0.0f) {
            const uint32_t q = f.id[k] << 5;
            const int pos = lower_bound32(s.sorted, q);
            if (pos < 32) {
                const uint32_t hit = s.sorted[pos];
                if ((hit >> 5) == f.id[k]) { known[k] = true; src[k] = (int)(hit & 31u); }
            }
        }
    }
    Texel<FMT> p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = Texel<FMT>::shfl(val, src[k]);
    __syncwarp();
    if (!active) return make_float4(0.f, 0.f, 0.f, 0.f);
    bool all_known = true;
    int N = 0;
    float Sw = 0.f, Swp[4] = {0.f, 0.f, 0.f, 0.f}, Sp[4] = {0.f, 0.f, 0.f, 0.f};
    int last = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!first[k] || dw[k] == 0.0f) continue;
        if (!known[k]) { all_known = false; continue; }
        ++N;
        last = k;
        Sw += dw[k];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            Swp[ch] = fmaf(dw[k], p[k].ch(ch), Swp[ch]);
            Sp[ch] += p[k].ch(ch);
        }
    }
    if (all_known) {
        // duplicates take their first occurrence's value; unknown corners have weight 0
        Texel<FMT> q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            q[k] = known[k] ? p[k] : Texel<FMT>::zero();
#pragma unroll
            for (int j = 0; j < k; ++j)
                if (f.id[j] == f.id[k] && known[j]) { q[k] = p[j]; break; }
        }
        return blend4<FMT>(q, f.w);
    }
    Texel<FMT> pl = p[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) if (k == last) pl = p[k];
    if (N == 1) return scaled<FMT>(pl);
    const float sc = Texel<FMT>::kScale;
    float c[4];
    if (wc) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) c[ch] = Swp[ch] / Sw * sc;
    } else {
        const float rest = (1.0f - Sw) / (float)N;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) c[ch] = fmaf(rest, Sp[ch], Swp[ch]) * sc;
    }
    return make_float4(c[0], c[1], c[2], c[3]);
}

template <int FMT, int MODE>
__global__ void __launch_bounds__(kWarps * 32) ctf_filter_kernel(const KArgs a) {
    __shared__ WarpSmem smem[kWarps];
    __shared__ __align__(16) float mlpw[FMT == FMT_MLP ? kMlpParams : 4];
    if constexpr (FMT == FMT_MLP) {
        for (int i = threadIdx.x; i < kMlpParams; i += blockDim.x) mlpw[i] = __ldg(a.tex.mlp + i);
        __syncthreads();
    }
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    WarpSmem &s = smem[warp];
    const bool debug = (a.flags & FLAG_DEBUG) != 0;
    const long long nwarps = (long long)gridDim.x * kWarps;

    for (long long w = (long long)blockIdx.x * kWarps + warp; w < a.total_waves; w += nwarps) {
        const int fr = (int)(w / a.wpf);
        const int rw = (int)(w - (long long)fr * a.wpf);
        const int wy = rw / a.nwx, wx = rw - wy * a.nwx;
        const int px = wx * 8 + (int)(lane & 7), py = wy * 4 + (int)(lane >> 3);
        const bool inframe = px < a.Wf && py < a.Hf;
        const size_t pix = (size_t)fr * (size_t)a.Wf * (size_t)a.Hf + (size_t)py * (size_t)a.Wf + (size_t)px;

        // ---- a1: load + classify
        float2 uv = make_float2(__int_as_float(0x7fc00000), 0.f);
        uint2 gr = make_uint2(0u, 0u);
        if (inframe) {
            uv = ld_stream_f2(a.uv + pix);
            if (a.grad) gr = ld_stream_u2(a.grad + pix);
        }
        const bool active = inframe && !isnan(uv.x);
        const unsigned A = __ballot_sync(FULL, active);
        const int na = __popc(A);
        if (na == 0) {
            if (inframe) st_stream_f4(a.out + pix, make_float4(0.f, 0.f, 0.f, 0.f));
            if (debug && inframe) {
                if (a.dbg_pid) a.dbg_pid[pix] = INVALID_ID;
                if (a.dbg_sel) a.dbg_sel[pix] = 0u;
            }
            if (lane == 0) a.rec[w] = ((MODE == MODE_COLLAB ? 0u : 0xFFu) << 8) | (1u << 26);
            continue;
        }
        bool mag_lane = true;
        if (a.grad) {
            const float2 g01 = __half22float2(*reinterpret_cast<const __half2 *>(&gr.x));
            const float2 g23 = __half22float2(*reinterpret_cast<const __half2 *>(&gr.y));
            const float rx = __fadd_rn(__fmul_rn(g01.x, g01.x), __fmul_rn(g01.y, g01.y));
            const float ry = __fadd_rn(__fmul_rn(g23.x, g23.x), __fmul_rn(g23.y, g23.y));
            mag_lane = (rx > ry ? rx : ry) <= 1.0f;  // R-20
        }
        const bool wave_mag = a.grad != nullptr && __all_sync(FULL, !active || mag_lane);

        // ---- a2: footprint
        const Foot f = footprint(uv, a);

        Texel<FMT> val = Texel<FMT>::zero();
        uint32_t prod = INVALID_ID;   // texel id this lane produced
        uint32_t selbits = 0u;
        float4 color = make_float4(0.f, 0.f, 0.f, 0.f);
        int n = 0xFF, evals = 0, path = 0;
        int run_fb = -1;

        if constexpr (MODE == MODE_4TAP) {
            path = PATH_4TAP;
            evals = 4 * na;
            if (active) {
                Texel<FMT> p[4];
                p[0] = produce<FMT>(a.tex, mlpw, f.xa, f.ya);
                p[1] = produce<FMT>(a.tex, mlpw, f.xb, f.ya);
                p[2] = produce<FMT>(a.tex, mlpw, f.xa, f.yb);
                p[3] = produce<FMT>(a.tex, mlpw, f.xb, f.yb);
                color = blend4<FMT>(p, f.w);
            }
        } else if constexpr (MODE == MODE_STF) {
            path = PATH_STF;
            run_fb = FB_STF;
        } else if constexpr (MODE == MODE_WC) {
            path = PATH_WC;
            run_fb = FB_WC;
        } else {
            // ---- a3: collect the exact unique set U and the canonical ranks
            const int minx = __reduce_min_sync(FULL, active ? f.xa : INT_MAX);
            const int maxx = __reduce_max_sync(FULL, active ? f.xb : INT_MIN);
            const int miny = __reduce_min_sync(FULL, active ? f.ya : INT_MAX);
            const int maxy = __reduce_max_sync(FULL, active ? f.yb : INT_MIN);
            const int bw = maxx - minx + 1, bh = maxy - miny + 1;
            const int lgP = bw <= 1 ? 0 : 32 - __clz(bw - 1);
            const bool fast = bw <= 32 && bh <= 128 && (bh << lgP) <= 128;
            int rho[4];
            if (fast) {
                // bit t = (y - miny) * P + (x - minx) of a <=128-bit AABB mask (rows never straddle words)
                const int t0 = ((f.ya - miny) << lgP) + (f.xa - minx);
                const int t2 = t0 + ((f.yb - f.ya) << lgP);
                const uint32_t dxs = (uint32_t)(f.xb - f.xa);
                const uint32_t pat = 1u | (dxs << 1);
                const int nwords = ((bh << lgP) + 31) >> 5;
                uint32_t B[4] = {0u, 0u, 0u, 0u};
                int pre[4] = {0, 0, 0, 0};
                n = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k < nwords) {
                        uint32_t m = 0u;
                        if (active) {
                            if ((t0 >> 5) == k) m |= pat << (t0 & 31);
                            if ((t2 >> 5) == k) m |= pat << (t2 & 31);
                        }
                        B[k] = __reduce_or_sync(FULL, m);
                        pre[k] = n;
                        n += __popc(B[k]);
                    }
                }
                auto rank = [&](int t) {
                    const int k = t >> 5;
                    const uint32_t bk = k == 0 ? B[0] : k == 1 ? B[1] : k == 2 ? B[2] : B[3];
                    const int pk = k == 0 ? pre[0] : k == 1 ? pre[1] : k == 2 ? pre[2] : pre[3];
                    return pk + __popc(bk & ((1u << (t & 31)) - 1u));
                };
                rho[0] = rank(t0);
                rho[1] = rho[0] + (int)dxs;
                rho[2] = rank(t2);
                rho[3] = rho[2] + (int)dxs;
                // producer table: rank -> (x, y) packed; lane j owns bit j of every word
                const unsigned lt = lanemask_lt();
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k < nwords && ((B[k] >> lane) & 1u)) {
                        const int r = pre[k] + __popc(B[k] & lt);
                        const uint32_t t = ((uint32_t)k << 5) | lane;
                        if (r < 32)
                            s.tbl[r] = ((uint32_t)(miny + (int)(t >> lgP)) << 16) |
                                       (uint32_t)(minx + (int)(t & ((1u << lgP) - 1u)));
                    }
                }
            } else {
                // slow path: sort the 128 (id << 7 | lane << 2 | corner) keys
                uint32_t key[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) key[k] = active ? ((f.id[k] << 7) | (lane << 2) | (uint32_t)k) : INVALID_ID;
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
                n = __shfl_sync(FULL, incl, 31);
                int run = incl - cnt;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    run += fl[k];
                    if (key[k] != INVALID_ID) {
                        const int r = run - 1;
                        s.rank_of[key[k] & 127u] = (uint8_t)r;
                        if (fl[k] && r < 32) {
                            const uint32_t id = key[k] >> 7;
                            const uint32_t y = id / (uint32_t)a.tex.W;
                            s.tbl[r] = (y << 16) | (id - y * (uint32_t)a.tex.W);
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 4; ++k) rho[k] = active ? (int)s.rank_of[lane * 4 + k] : 0;
            }
            __syncwarp();
            // ---- a4: decide
            const bool exact = n <= na && !(a.flags & FLAG_FORCE_FALLBACK);
            if (exact) {
                path = PATH_EXACT;
                evals = n;
                const bool full = A == FULL;
                const int ar = __popc(A & lanemask_lt());
                if (!full) {
                    if (active) s.lane_of_rank[ar] = (uint8_t)lane;
                    __syncwarp();
                }
                // ---- a5: active rank r < n produces U[r] (lane h(r, A))
                const bool producer = active && ar < n;
                if (producer) {
                    const uint32_t xy = s.tbl[ar];
                    val = produce<FMT>(a.tex, mlpw, xy & 0xffffu, xy >> 16);
                    prod = (xy >> 16) * (uint32_t)a.tex.W + (xy & 0xffffu);
                }
                // ---- a6: gather from lanes h(rho_k, A) and blend
                int src[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    src[k] = active ? (full ? rho[k] : (int)s.lane_of_rank[rho[k]]) : (int)lane;
                }
                Texel<FMT> p[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) p[k] = Texel<FMT>::shfl(val, src[k]);
                if (active) color = blend4<FMT>(p, f.w);
                if (debug && a.dbg_unread) {
                    int bad = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) bad += (active && !__shfl_sync(FULL, producer, src[k])) ? 1 : 0;
                    if (bad) atomicAdd(a.dbg_unread, (unsigned)bad);
                }
            } else {
                run_fb = a.fallback;
                path = PATH_FB_STF + a.fallback;
            }
        }

        // ---- a7: fallbacks (and the pure STF / WC modes)
        if (MODE != MODE_4TAP && run_fb >= 0) {
            const uint4 rr = philox4x32_10(make_uint4((uint32_t)px, (uint32_t)py, a.frame_index + (uint32_t)fr, 0u),
                                           a.seed_lo, a.seed_hi);
            const int ksel = stf_corner(f, rr);
            selbits = active ? (uint32_t)ksel : 0u;
            if (run_fb == FB_STF) {
                evals = na;
                if (active) {
                    prod = corner_id(f, ksel);
                    val = produce<FMT>(a.tex, mlpw, corner_x(f, ksel), corner_y(f, ksel));
                    color = scaled<FMT>(val);
                }
            } else if (run_fb == FB_WC || run_fb == FB_C) {
                evals = na;
                if (active) {
                    prod = corner_id(f, ksel);
                    val = produce<FMT>(a.tex, mlpw, corner_x(f, ksel), corner_y(f, ksel));
                }
                color = fallback_gather<FMT>(f, active, prod, val, run_fb == FB_WC, s);
            } else {
                // C+ (P:485-518): (1) planned STF texels, deduplicated and ranked ascending
                const uint32_t pid = corner_id(f, ksel);
                const uint32_t sk = warp_sort32(active ? ((pid << 5) | lane) : INVALID_ID);
                const uint32_t skp = __shfl_up_sync(FULL, sk, 1);
                const bool firstp = sk != INVALID_ID && (lane == 0 || (sk >> 5) != (skp >> 5));
                const unsigned F = __ballot_sync(FULL, firstp);
                const int np = __popc(F);
                if (firstp) s.tbl[__popc(F & lanemask_lt())] = sk >> 5;
                if ((int)lane >= np) s.tbl[lane] = INVALID_ID;
                const int ar = __popc(A & lanemask_lt());
                if (active) s.lane_of_rank[ar] = (uint8_t)lane;
                __syncwarp();
                // (2) active ranks < n_p produce the planned texels
                bool spare = false;
                int l = (int)lane;
                if (active) {
                    if (ar < np) {
                        prod = s.tbl[ar];
                        const uint32_t y = prod / (uint32_t)a.tex.W;
                        val = produce<FMT>(a.tex, mlpw, prod - y * (uint32_t)a.tex.W, y);
                    } else {
                        spare = true;
                        l = (int)s.lane_of_rank[eq2_lane_rank(ar, np, na)];  // (3) Eq. 2
                        selbits |= (1u << 5) | ((uint32_t)l << 8);
                    }
                }
                // spare lanes fetch the served lane's footprint
                Foot g;
                g.xa = __shfl_sync(FULL, f.xa, l);
                g.xb = __shfl_sync(FULL, f.xb, l);
                g.ya = __shfl_sync(FULL, f.ya, l);
                g.yb = __shfl_sync(FULL, f.yb, l);
                g.s = __shfl_sync(FULL, f.s, l);
                g.t = __shfl_sync(FULL, f.t, l);
                if (spare) {
                    make_ids(g, a.tex.W);
                    make_weights(g);
                    // candidates: distinct nonzero-weight texels of l's footprint not in P (R-18 v)
                    bool cand[4];
                    float cw[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) { cand[k] = true; cw[k] = g.w[k]; }
#pragma unroll
                    for (int k = 1; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < k; ++j)
                            if (cand[j] && cand[k] && g.id[j] == g.id[k]) {
                                cand[k] = false;
                                cw[j] = __fadd_rn(cw[j], g.w[k]);
                            }
                    float wsum = 0.0f;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (cand[k] && cw[k] != 0.0f) {
                            const int pos = lower_bound32(s.tbl, g.id[k]);
                            if (pos < 32 && s.tbl[pos] == g.id[k]) cand[k] = false;
                        } else {
                            cand[k] = false;
                        }
                        if (cand[k]) wsum = __fadd_rn(wsum, cw[k]);
                    }
                    if (cand[0] || cand[1] || cand[2] || cand[3]) {
                        const float target = __fmul_rn(unit24(rr.z), wsum);
                        float cum = 0.0f;
                        int pick = -1, lastc = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (!cand[k]) continue;
                            lastc = k;
                            cum = __fadd_rn(cum, cw[k]);
                            if (pick < 0 && cum > target) pick = k;
                        }
                        if (pick < 0) pick = lastc;
                        prod = corner_id(g, pick);
                        val = produce<FMT>(a.tex, mlpw, corner_x(g, pick), corner_y(g, pick));
                        selbits |= ((uint32_t)pick << 2) | (1u << 4);
                    }
                }
                __syncwarp();
                evals = __popc(__ballot_sync(FULL, active && prod != INVALID_ID));
                color = fallback_gather<FMT>(f, active, prod, val, false, s);
            }
        }

        // ---- outputs
        if (inframe) st_stream_f4(a.out + pix, color);
        if (debug && inframe) {
            if (a.dbg_pid) a.dbg_pid[pix] = (MODE == MODE_4TAP) ? INVALID_ID : prod;
            if (a.dbg_sel) a.dbg_sel[pix] = selbits;
        }
        // ---- a8: per-wave record
        if (lane == 0)
            a.rec[w] = (uint32_t)(evals & 0xFF) | ((uint32_t)(n & 0xFF) << 8) | ((uint32_t)na << 16) |
                       ((uint32_t)path << 22) | ((uint32_t)wave_mag << 25) | ((uint32_t)(na < 32) << 26);
        __syncwarp();
    }
}

template <int FMT, int MODE>
static cudaError_t launch_one(const KArgs &k, cudaStream_t stream) {
    auto kern = ctf_filter_kernel<FMT, MODE>;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, 0);
    if (e != cudaSuccess) return e;
    const long long need = (k.total_waves + kWarps - 1) / kWarps;
    long long grid = (long long)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kWarps * 32, 0, stream>>>(k);
    return cudaGetLastError();
}

template <int FMT>
static cudaError_t launch_fmt(const KArgs &k, int mode, cudaStream_t stream) {
    switch (mode) {
    case MODE_4TAP: return launch_one<FMT, MODE_4TAP>(k, stream);
    case MODE_STF: return launch_one<FMT, MODE_STF>(k, stream);
    case MODE_WC: return launch_one<FMT, MODE_WC>(k, stream);
    default: return launch_one<FMT, MODE_COLLAB>(k, stream);
    }
}

#ifndef CTF_TU_FMT
#error "compile ctf_filter.cu with -DCTF_TU_FMT=1 (BC1) or =2 (latent MLP)"
#endif
#if CTF_TU_FMT == 1
cudaError_t launch_filter_bc1(const LaunchArgs &a, cudaStream_t stream) {
#else
cudaError_t launch_filter_mlp(const LaunchArgs &a, cudaStream_t stream) {
#endif
    KArgs k;
    k.tex.W = a.W;
    k.tex.H = a.H;
    k.tex.bc1 = reinterpret_cast<const uint2 *>(a.tex_data);
    k.tex.latent = reinterpret_cast<const uint4 *>(a.tex_data);
    k.tex.mlp = a.mlp;
    k.uv = reinterpret_cast<const float2 *>(a.uv);
    k.grad = reinterpret_cast<const uint2 *>(a.grad);
    k.out = reinterpret_cast<float4 *>(a.out);
    k.rec = a.rec;
    k.dbg_pid = a.dbg_pid;
    k.dbg_sel = a.dbg_sel;
    k.dbg_unread = a.dbg_unread;
    k.Wf = a.Wf;
    k.Hf = a.Hf;
    k.nwx = (a.Wf + 7) / 8;
    k.wpf = k.nwx * ((a.Hf + 3) / 4);
    k.total_waves = (long long)k.wpf * a.frames;
    k.Wflt = (float)a.W;
    k.Hflt = (float)a.H;
    k.fallback = a.fallback;
    k.flags = a.flags;
    k.frame_index = a.frame_index;
    k.seed_lo = (uint32_t)a.seed;
    k.seed_hi = (uint32_t)(a.seed >> 32);
#if CTF_TU_FMT == 1
    return launch_fmt<FMT_BC1>(k, a.mode, stream);
#else
    return launch_fmt<FMT_MLP>(k, a.mode, stream);
#endif
}

}  // namespace ctf
