/*
 * ctf_oracle.c — CPU ORACLE for collaborative texture filtering (CTF),
 * arXiv 2506.17770 ("Collaborative Texture Filtering").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2506_17770_b200/csrc); the only thing both see is the input bytes
 * written by synthetic/.
 *
 * It is deliberately plain and slow: one wave at a time, brute force where a
 * plain definition exists (the exact unique-texel set is a sort + unique; the
 * exact-path colour is plain 4-tap bilinear), the paper's algorithm step by
 * step elsewhere (fallbacks C / C+, Eq. 1, Eq. 2).  Colours are fp64.
 * Quantities that decide an integer (texel coordinates from floor(), STF and
 * C+ selections, the magnified class) are computed in fp32 with the op order
 * fixed in DESIGN.md "Readings", because the parity rule takes such decisions
 * in the kernel's precision.  Compile with -ffp-contract=off (no FMA
 * contraction) and without -ffast-math.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * R-n = reading n in DESIGN.md (SURVEY §8(c) row cN).
 *
 * Parity pins (tests/test_oracle_pins.py): every function below is pinned by
 * the paper's worked examples, closed forms or brute force except
 *   - bc1 decode (R-9) and the latent-MLP decode (R-10): our synthetic
 *     formats — pinned by hand-decoded vectors / an independent numpy fp64
 *     evaluation, never by the paper ("parity unpinned" by the paper);
 *   - the WC stand-in rule (R-16) and the C+ selection law (R-18 v):
 *     pinned only by their special cases ("parity unpinned" beyond those).
 * Bicubic filters (wave_bicubic, R-24..R-28) are pinned in
 * tests/test_oracle_bicubic.py by the kernels' closed-form moments, texel-centre
 * interpolation / smoothing, linear reproduction on a ramp, brute-force unique
 * sets and the expectations of the stochastic estimators; the C+ selection law
 * for bicubic (R-18 v with |w|) is, as for bilinear, pinned only by its special
 * cases.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define INVALID_ID 0xFFFFFFFFu

/* modes / fallbacks / flags as numbered in DESIGN.md (the boundary's values) */
enum { M_4TAP = 0, M_STF = 1, M_WC = 2, M_COLLAB = 3, M_BOX = 4, M_MASK16 = 5, M_MASK11 = 6 };
enum { FB_STF = 0, FB_WC = 1, FB_C = 2, FB_CPLUS = 3 };
enum { FL_DEBUG = 1u, FL_FORCE_FALLBACK = 2u };
enum { PATH_EXACT = 0, PATH_FB_STF = 1, PATH_FB_WC = 2, PATH_FB_C = 3, PATH_FB_CPLUS = 4,
       PATH_4TAP = 5, PATH_STF = 6, PATH_WC = 7 };
enum { FMT_BC1 = 1, FMT_LATENT_MLP = 2 };

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11 / Random123) — R-11.  The paper only
 * asks for a random STF choice; the generator is ours.           */
/* ------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* uniform in [0,1) from the top 24 bits: exact in fp32 and fp64 (R-11) */
static double unit24(uint32_t r) { return (double)(r >> 8) * (1.0 / 16777216.0); }

static void pixel_uniforms(int px, int py, uint32_t frame, uint64_t seed, double u[4])
{
    uint32_t ctr[4] = { (uint32_t)px, (uint32_t)py, frame, 0u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t r[4];
    oracle_philox4x32_10(ctr, key, r);
    for (int k = 0; k < 4; ++k) u[k] = unit24(r[k]);
}

/* ------------------------------------------------------------------------- */
/* IEEE half -> float (exact), written out from the binary16 definition.     */
/* ------------------------------------------------------------------------- */
static float half_to_float(uint16_t h)
{
    uint32_t sign = (uint32_t)(h >> 15) & 1u, ex = (uint32_t)(h >> 10) & 31u, man = h & 1023u;
    float mag;
    if (ex == 0) mag = ldexpf((float)man, -24);               /* subnormal / zero */
    else if (ex == 31) mag = man ? NAN : INFINITY;
    else mag = ldexpf((float)(man + 1024u), (int)ex - 25);
    return sign ? -mag : mag;
}

/* ------------------------------------------------------------------------- */
/* Texel production (the "evaluation" of step 2).                  */
/* ------------------------------------------------------------------------- */
typedef struct {
    int format, W, H;
    const uint8_t *bc1;          /* FMT_BC1: (H/4)*(W/4) blocks of 8 bytes       */
    const uint16_t *latent;      /* FMT_LATENT_MLP: half bits [H/4][W/4][8]      */
    const float *mlp;            /* packed W1[32][12] b1 W2[32][32] b2 W3[4][32] b3 */
} tex_t;

/* R-9: synthetic BC1-style block decode -> 4 channel bytes (0..255).
 * block = ((y>>2)*(W>>2) + (x>>2)); c0 = u16@0, c1 = u16@2, idx = u32@4;
 * code = (idx >> 2*(4*(y&3) + (x&3))) & 3; RGB565 -> 888 by bit replication;
 * c0 > c1: {c0, c1, (2c0+c1)/3, (c0+2c1)/3}, alpha 255;
 * else   : {c0, c1, (c0+c1)/2, transparent black}; integer division truncates. */
void oracle_bc1_texel(const uint8_t *blocks, int W, int x, int y, uint8_t rgba[4])
{
    const uint8_t *b = blocks + 8 * ((size_t)(y >> 2) * (size_t)(W >> 2) + (size_t)(x >> 2));
    uint32_t c0 = (uint32_t)b[0] | ((uint32_t)b[1] << 8);
    uint32_t c1 = (uint32_t)b[2] | ((uint32_t)b[3] << 8);
    uint32_t idx = (uint32_t)b[4] | ((uint32_t)b[5] << 8) | ((uint32_t)b[6] << 16) | ((uint32_t)b[7] << 24);
    uint32_t code = (idx >> (2 * (4 * (y & 3) + (x & 3)))) & 3u;
    int e0[3], e1[3];
    int r0 = (c0 >> 11) & 31, g0 = (c0 >> 5) & 63, b0 = c0 & 31;
    int r1 = (c1 >> 11) & 31, g1 = (c1 >> 5) & 63, b1 = c1 & 31;
    e0[0] = (r0 << 3) | (r0 >> 2); e0[1] = (g0 << 2) | (g0 >> 4); e0[2] = (b0 << 3) | (b0 >> 2);
    e1[0] = (r1 << 3) | (r1 >> 2); e1[1] = (g1 << 2) | (g1 >> 4); e1[2] = (b1 << 3) | (b1 >> 2);
    int out[4];
    for (int c = 0; c < 3; ++c) {
        if (code == 0) out[c] = e0[c];
        else if (code == 1) out[c] = e1[c];
        else if (c0 > c1) out[c] = (code == 2) ? (2 * e0[c] + e1[c]) / 3 : (e0[c] + 2 * e1[c]) / 3;
        else out[c] = (code == 2) ? (e0[c] + e1[c]) / 2 : 0;
    }
    out[3] = (c0 > c1 || code != 3) ? 255 : 0;
    for (int c = 0; c < 4; ++c) rgba[c] = (uint8_t)out[c];
}

/* R-10: latent + MLP decode (NTC-style inference-on-sample), fp64.
 * Latent grid (W/4)x(H/4)x8 sampled at ((x-1.5)/4, (y-1.5)/4) with clamped
 * bilinear interpolation; 4 positional features; MLP 12->32->32->4 with
 * ReLU, ReLU, clamp[0,1]. */
void oracle_mlp_texel(const uint16_t *latent, const float *mlp, int W, int H, int x, int y, double rgba[4])
{
    int lw = W / 4, lh = H / 4;
    double gx = (x - 1.5) / 4.0, gy = (y - 1.5) / 4.0;
    double fx0 = floor(gx), fy0 = floor(gy);
    double fx = gx - fx0, fy = gy - fy0;
    int ix[2] = { (int)fx0, (int)fx0 + 1 }, iy[2] = { (int)fy0, (int)fy0 + 1 };
    for (int k = 0; k < 2; ++k) {
        ix[k] = ix[k] < 0 ? 0 : (ix[k] > lw - 1 ? lw - 1 : ix[k]);
        iy[k] = iy[k] < 0 ? 0 : (iy[k] > lh - 1 ? lh - 1 : iy[k]);
    }
    double wgt[4] = { (1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy };
    double in[12];
    for (int c = 0; c < 8; ++c) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k) {
            int xx = ix[k & 1], yy = iy[k >> 1];
            acc += wgt[k] * (double)half_to_float(latent[((size_t)yy * lw + xx) * 8 + c]);
        }
        in[c] = acc;
    }
    in[8] = ((x & 3) - 1.5) / 2.0;
    in[9] = ((y & 3) - 1.5) / 2.0;
    in[10] = ((x >> 2) & 1) - 0.5;
    in[11] = ((y >> 2) & 1) - 0.5;
    const float *W1 = mlp, *b1 = W1 + 32 * 12, *W2 = b1 + 32, *b2 = W2 + 32 * 32, *W3 = b2 + 32, *b3 = W3 + 4 * 32;
    double h1[32], h2[32];
    for (int j = 0; j < 32; ++j) {
        double acc = b1[j];
        for (int k = 0; k < 12; ++k) acc += (double)W1[j * 12 + k] * in[k];
        h1[j] = acc > 0 ? acc : 0;
    }
    for (int j = 0; j < 32; ++j) {
        double acc = b2[j];
        for (int k = 0; k < 32; ++k) acc += (double)W2[j * 32 + k] * h1[k];
        h2[j] = acc > 0 ? acc : 0;
    }
    for (int j = 0; j < 4; ++j) {
        double acc = b3[j];
        for (int k = 0; k < 32; ++k) acc += (double)W3[j * 32 + k] * h2[k];
        rgba[j] = acc < 0 ? 0 : (acc > 1 ? 1 : acc);
    }
}

/* produce texel `id` (= y*W + x) -> fp64 RGBA in [0,1] */
static void produce(const tex_t *t, uint32_t id, double rgba[4])
{
    int x = (int)(id % (uint32_t)t->W), y = (int)(id / (uint32_t)t->W);
    if (t->format == FMT_BC1) {
        uint8_t b[4];
        oracle_bc1_texel(t->bc1, t->W, x, y, b);
        for (int c = 0; c < 4; ++c) rgba[c] = (double)b[c] / 255.0;
    } else {
        oracle_mlp_texel(t->latent, t->mlp, t->W, t->H, x, y, rgba);
    }
}

/* ------------------------------------------------------------------------- */
/* Footprint and weights — R-2, R-3.      */
/* ------------------------------------------------------------------------- */
typedef struct {
    int active;
    int x[2], y[2];        /* clamped texel columns {x0, x0+1} and rows {y0, y0+1} (R-2 i) */
    uint32_t id[4];        /* corners UL, UR, LL, LR: id = y*W + x (R-3 order) */
    float s, t;            /* fp32 fractional position (decides integer coords) */
    float w32[4];          /* fp32 weights, used ONLY for the C+ pick decision (R-18 v) */
    double w[4];           /* fp64 weights for colour */
    int magnified;         /* R-20 */
} lane_t;

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* exported for the pins: footprint of one uv -> ids, s, t */
void oracle_footprint(float u, float v, int W, int H, uint32_t id[4], float st[2])
{
    /* R-2: u, v clamped to [0, 1] (clamp-to-edge addressing; a NaN v maps to 0);
     * fx = fma(u, W, -0.5) with ONE fp32 rounding (the listing's uv * txDim - 0.5 as a
     * fused multiply-add); x0 = floor(fx); s = fx - x0 (exact in fp32).              */
    float uc = fminf(fmaxf(u, 0.0f), 1.0f);
    float vc = fminf(fmaxf(v, 0.0f), 1.0f);
    float fx = fmaf(uc, (float)W, -0.5f), fy = fmaf(vc, (float)H, -0.5f);
    float flx = floorf(fx), fly = floorf(fy);
    int x0 = (int)flx, y0 = (int)fly;
    st[0] = fx - flx;
    st[1] = fy - fly;
    int xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
    int ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
    id[0] = (uint32_t)ya * (uint32_t)W + (uint32_t)xa;
    id[1] = (uint32_t)ya * (uint32_t)W + (uint32_t)xb;
    id[2] = (uint32_t)yb * (uint32_t)W + (uint32_t)xa;
    id[3] = (uint32_t)yb * (uint32_t)W + (uint32_t)xb;
}

static void make_lane(lane_t *L, const float *uv, const uint16_t *grad, int W, int H)
{
    float st[2];
    oracle_footprint(uv[0], uv[1], W, H, L->id, st);
    L->s = st[0];
    L->t = st[1];
    /* fp64 weights (R-3): ((1-s)(1-t), s(1-t), (1-s)t, st), order UL, UR, LL, LR */
    double s = st[0], t = st[1];
    L->w[0] = (1.0 - s) * (1.0 - t);
    L->w[1] = s * (1.0 - t);
    L->w[2] = (1.0 - s) * t;
    L->w[3] = s * t;
    /* fp32 weights, each product rounded once, for fp32 decisions only */
    float a = 1.0f - L->s, b = 1.0f - L->t;
    L->w32[0] = a * b;
    L->w32[1] = L->s * b;
    L->w32[2] = a * L->t;
    L->w32[3] = L->s * L->t;
    /* R-20: rho^2 = max(Jxx^2 + Jyx^2, Jxy^2 + Jyy^2) in fp32; magnified <=> rho^2 <= 1.
     * The squares of fp16 values are exact in fp32, so each sum has one rounding. */
    L->magnified = 0;
    if (grad) {
        float g0 = half_to_float(grad[0]), g1 = half_to_float(grad[1]);
        float g2 = half_to_float(grad[2]), g3 = half_to_float(grad[3]);
        volatile float a0 = g0 * g0, a1 = g1 * g1, a2 = g2 * g2, a3 = g3 * g3;
        float rx = a0 + a1, ry = a2 + a3;
        float r2 = rx > ry ? rx : ry;
        L->magnified = (r2 <= 1.0f);
    }
}

/* ------------------------------------------------------------------------- */
/* h(i, B): position of the i-th set bit (Fig. 2);      */
/* h^-1(t, B): number of set bits below t.  Plain loops.         */
/* ------------------------------------------------------------------------- */
int oracle_h(uint32_t i, uint32_t B)
{
    for (int bit = 0; bit < 32; ++bit)
        if ((B >> bit) & 1u) { if (i == 0) return bit; --i; }
    return -1;
}

int oracle_h_inv(int t, uint32_t B)
{
    int c = 0;
    for (int bit = 0; bit < t; ++bit) c += (B >> bit) & 1u;
    return c;
}

/* Eq. 2, generalised to a active lanes (R-18 iv):
 * l = round_half_up((a-1)(c-n) / (a-1-n)) for n < a-1; l = 0 when n = a-1. */
int oracle_eq2(int c, int n, int a)
{
    if (n >= a - 1) return 0;
    long num = 2L * (a - 1) * (c - n) + (a - 1 - n);
    long den = 2L * (a - 1 - n);
    return (int)(num / den);
}

/* ------------------------------------------------------------------------- */
/* per-wave helpers                                                          */
/* ------------------------------------------------------------------------- */
static int cmp_u32(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : (x > y);
}

/* sort + unique; returns count, list in ascending order (R-5) */
static int sort_unique(uint32_t *v, int n)
{
    qsort(v, (size_t)n, sizeof(uint32_t), cmp_u32);
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (m == 0 || v[m - 1] != v[i]) v[m++] = v[i];
    return m;
}

static void blend_exact(const tex_t *tex, const lane_t *L, double c[4])
{
    /* plain 4-tap bilinear of the produced texels (R-8) */
    for (int ch = 0; ch < 4; ++ch) c[ch] = 0.0;
    for (int k = 0; k < 4; ++k) {
        double p[4];
        produce(tex, L->id[k], p);
        for (int ch = 0; ch < 4; ++ch) c[ch] += L->w[k] * p[ch];
    }
}

static int in_list(const uint32_t *list, int n, uint32_t id)
{
    for (int i = 0; i < n; ++i) if (list[i] == id) return 1;
    return 0;
}

/* Eq. 1 over the known set K_L (R-14/R-15); wc != 0 -> R-16. */
static void blend_fallback(const tex_t *tex, const lane_t *L, const uint32_t *produced, int nprod,
                           int wc, double c[4])
{
    /* distinct footprint texels in first-occurrence corner order, merged weights (R-14) */
    uint32_t did[4]; double dw[4]; int nd = 0;
    for (int k = 0; k < 4; ++k) {
        int j;
        for (j = 0; j < nd; ++j) if (did[j] == L->id[k]) break;
        if (j == nd) { did[nd] = L->id[k]; dw[nd] = 0.0; ++nd; }
        dw[j] += L->w[k];
    }
    int all_known = 1, N = 0;
    double Swp[4] = { 0, 0, 0, 0 }, Sp[4] = { 0, 0, 0, 0 }, Sw = 0.0, plast[4] = { 0, 0, 0, 0 };
    for (int j = 0; j < nd; ++j) {
        if (dw[j] == 0.0) continue;               /* only nonzero filter weights */
        if (!in_list(produced, nprod, did[j])) { all_known = 0; continue; }
        double p[4];
        produce(tex, did[j], p);
        for (int ch = 0; ch < 4; ++ch) { Swp[ch] += dw[j] * p[ch]; Sp[ch] += p[ch]; plast[ch] = p[ch]; }
        Sw += dw[j];
        ++N;
    }
    if (all_known) { blend_exact(tex, L, c); return; }
    if (N == 1) { for (int ch = 0; ch < 4; ++ch) c[ch] = plast[ch]; return; }
    for (int ch = 0; ch < 4; ++ch) {
        if (wc) c[ch] = Swp[ch] / Sw;                          /* R-16 */
        else c[ch] = Swp[ch] + (1.0 - Sw) * Sp[ch] / N;       /* Eq. 1 */
    }
}

/* STF corner choice (R-12): dx = (u0 < s), dy = (u1 < t) */
static int stf_corner(const lane_t *L, const double u[4])
{
    int dx = u[0] < (double)L->s;
    int dy = u[1] < (double)L->t;
    return dx + 2 * dy;
}

/* ------------------------------------------------------------------------- */
/* One wave (8x4 pixels, lane = 8*ly + lx; P:266-268, S:79 — R-1).           */
/* ------------------------------------------------------------------------- */
typedef struct {
    const tex_t *tex;
    const float *uv; const uint16_t *grad;
    int Wf, Hf;
    int mode, fallback; unsigned flags; uint64_t seed; uint32_t frame;
    double *out; uint32_t *rec; uint32_t *produced_id; uint32_t *selection;
} frame_t;

static void wave(const frame_t *F, int wx, int wy)
{
    const tex_t *tex = F->tex;
    lane_t L[32];
    int px[32], py[32], inframe[32];
    uint32_t A = 0;
    for (int lane = 0; lane < 32; ++lane) {
        px[lane] = wx * 8 + (lane & 7);
        py[lane] = wy * 4 + (lane >> 3);
        inframe[lane] = px[lane] < F->Wf && py[lane] < F->Hf;
        memset(&L[lane], 0, sizeof(lane_t));
        if (!inframe[lane]) continue;
        size_t pix = (size_t)py[lane] * F->Wf + px[lane];
        const float *uvp = F->uv + 2 * pix;
        if (isnan(uvp[0])) continue;                                   /* uncovered */
        L[lane].active = 1;
        A |= 1u << lane;
        make_lane(&L[lane], uvp, F->grad ? F->grad + 4 * pix : NULL, tex->W, tex->H);
    }
    int a = __builtin_popcount(A);
    int nwx = (F->Wf + 7) / 8;
    uint32_t *rec = &F->rec[(size_t)wy * nwx + wx];

    /* outputs default: uncovered -> 0, debug -> none */
    double col[32][4];
    uint32_t prod[32], sel[32];
    for (int lane = 0; lane < 32; ++lane) {
        for (int ch = 0; ch < 4; ++ch) col[lane][ch] = 0.0;
        prod[lane] = INVALID_ID; sel[lane] = 0;
    }
    int magnified = 0;
    if (F->grad && a > 0) {
        magnified = 1;
        for (int lane = 0; lane < 32; ++lane) if (L[lane].active && !L[lane].magnified) magnified = 0;
    }

    /* lanes in active order: act[r] = h(r, A) */
    int act[32];
    for (int r = 0; r < a; ++r) act[r] = oracle_h((uint32_t)r, A);

    double u[32][4];
    for (int lane = 0; lane < 32; ++lane)
        if (L[lane].active) pixel_uniforms(px[lane], py[lane], F->frame, F->seed, u[lane]);

    int n = 0xFF, evals = 0, path = 0;
    int run_fallback = -1;   /* which fallback estimator runs, -1 = none */

    if (F->mode == M_4TAP) {
        path = PATH_4TAP;
        for (int lane = 0; lane < 32; ++lane) if (L[lane].active) blend_exact(tex, &L[lane], col[lane]);
        evals = 4 * a;                          /* classic bilinear: 4 evaluations per pixel */
    } else if (F->mode == M_STF) {
        path = PATH_STF; run_fallback = FB_STF;
    } else if (F->mode == M_WC) {
        path = PATH_WC; run_fallback = FB_WC;
    } else {
        /* step 1 "collect": exact unique set U over active footprints (R-4/R-5) */
        uint32_t U[128];
        int m = 0;
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) for (int k = 0; k < 4; ++k) U[m++] = L[lane].id[k];
        n = sort_unique(U, m);
        /* wave AABB of the clamped footprints */
        int minx = 1 << 30, maxx = -1, miny = 1 << 30, maxy = -1;
        for (int lane = 0; lane < 32; ++lane) {
            if (!L[lane].active) continue;
            int xa = (int)(L[lane].id[0] % (uint32_t)tex->W), ya = (int)(L[lane].id[0] / (uint32_t)tex->W);
            int xb = (int)(L[lane].id[3] % (uint32_t)tex->W), yb = (int)(L[lane].id[3] / (uint32_t)tex->W);
            if (xa < minx) minx = xa;
            if (ya < miny) miny = ya;
            if (xb > maxx) maxx = xb;
            if (yb > maxy) maxy = yb;
        }
        int bw = 0, bh = 0, ok = 0;
        if (a > 0) {
            bw = maxx - minx + 1;
            bh = maxy - miny + 1;
            if (F->mode == M_BOX) ok = bw * bh <= a;                              /* P:345-346 + remap */
            else if (F->mode == M_MASK16) ok = bw <= 16 && bh <= 16 && n <= a;
            else if (F->mode == M_MASK11) ok = bw <= 11 && bh <= 11 && n <= a;
            else ok = n <= a;                                                     /* List, R-6 */
        }
        if (a > 0 && ok && !(F->flags & FL_FORCE_FALLBACK)) {
            path = PATH_EXACT;
            if (F->mode == M_BOX) {
                /* Box: active rank i < bw*bh produces AABB texel (i mod bw, i div bw)
                 * (LaneIdxToCoord P:1069-1076, with edge remapping P:1381) */
                for (int i = 0; i < bw * bh; ++i)
                    prod[act[i]] = (uint32_t)(miny + i / bw) * (uint32_t)tex->W + (uint32_t)(minx + i % bw);
                evals = bw * bh;
            } else {
                /* step 2: rank r is produced by lane h(r, A) (R-7) */
                for (int r = 0; r < n; ++r) prod[act[r]] = U[r];
                evals = n;
            }
            /* step 3: each lane gathers its 4 texels; result = plain bilinear (R-8) */
            for (int lane = 0; lane < 32; ++lane) if (L[lane].active) blend_exact(tex, &L[lane], col[lane]);
        } else {
            run_fallback = F->fallback;
            path = PATH_FB_STF + F->fallback;
        }
    }

    if (run_fallback == FB_STF) {
        /* one-tap STF (Pharr 2024): colour = selected texel */
        for (int lane = 0; lane < 32; ++lane) {
            if (!L[lane].active) continue;
            int k = stf_corner(&L[lane], u[lane]);
            sel[lane] = (uint32_t)k;
            prod[lane] = L[lane].id[k];
            produce(tex, prod[lane], col[lane]);
        }
        evals = a;
    } else if (run_fallback == FB_WC || run_fallback == FB_C) {
        /* every lane produces its STF texel ... */
        uint32_t plist[32]; int np = 0;
        for (int lane = 0; lane < 32; ++lane) {
            if (!L[lane].active) continue;
            int k = stf_corner(&L[lane], u[lane]);
            sel[lane] = (uint32_t)k;
            prod[lane] = L[lane].id[k];
            plist[np++] = prod[lane];
        }
        /* ... and filters with the unique in-footprint texels of the wave (Eq. 1 / R-16) */
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) blend_fallback(tex, &L[lane], plist, np, run_fallback == FB_WC, col[lane]);
        evals = a;
    } else if (run_fallback == FB_CPLUS) {
        /* C+ (P:485-518).  (1) planned STF texels, deduplicated (R-17) */
        uint32_t P[32]; int np = 0;
        for (int lane = 0; lane < 32; ++lane) {
            if (!L[lane].active) continue;
            int k = stf_corner(&L[lane], u[lane]);
            sel[lane] = (uint32_t)k;
            P[np++] = L[lane].id[k];
        }
        np = sort_unique(P, np);
        uint32_t produced[32]; int nprod = 0;
        /* (2) the first n_p active lanes produce the planned texels, rank i -> lane h(i, A) */
        for (int i = 0; i < np && i < a; ++i) { prod[act[i]] = P[i]; produced[nprod++] = P[i]; }
        /* (3) spare lanes (active ranks j in [n_p, a-1]) serve lane l from Eq. 2 (R-18) */
        for (int j = np; j < a; ++j) {
            int c = act[j];
            int l = act[oracle_eq2(j, np, a)];
            sel[c] |= (1u << 5) | ((uint32_t)l << 8);
            const lane_t *Ll = &L[l];
            /* candidates: distinct nonzero-weight texels of l's footprint not in P,
             * first-occurrence corner order, fp32 merged weights (R-18 v) */
            uint32_t cid[4]; float cw[4]; int ck[4]; int nc = 0;
            for (int k = 0; k < 4; ++k) {
                int q;
                for (q = 0; q < nc; ++q) if (cid[q] == Ll->id[k]) break;
                if (q == nc) { cid[nc] = Ll->id[k]; cw[nc] = 0.0f; ck[nc] = k; ++nc; }
                cw[q] = cw[q] + Ll->w32[k];
            }
            uint32_t fid[4]; float fw[4]; int fk[4]; int nf = 0;
            for (int q = 0; q < nc; ++q) {
                if (cw[q] == 0.0f) continue;
                if (in_list(P, np, cid[q])) continue;
                fid[nf] = cid[q]; fw[nf] = cw[q]; fk[nf] = ck[q]; ++nf;
            }
            if (nf == 0) continue;                                   /* produce nothing */
            /* selection proportional to weight, decided in fp32 (parity rule) */
            float wsum = 0.0f;
            for (int q = 0; q < nf; ++q) wsum = wsum + fw[q];
            volatile float target = (float)u[c][2] * wsum;
            int pick = nf - 1;
            float cum = 0.0f;
            for (int q = 0; q < nf; ++q) {
                cum = cum + fw[q];
                if (cum > target) { pick = q; break; }
            }
            prod[c] = fid[pick];
            produced[nprod++] = fid[pick];
            sel[c] |= ((uint32_t)fk[pick] << 2) | (1u << 4);
        }
        /* (4) every lane filters with Eq. 1 over the produced set */
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) blend_fallback(tex, &L[lane], produced, nprod, 0, col[lane]);
        evals = nprod;
    }

    if (a == 0) { evals = 0; path = 0; if (F->mode >= M_COLLAB) n = 0; }
    *rec = (uint32_t)(evals & 0xFF) | ((uint32_t)(n & 0xFF) << 8) | ((uint32_t)a << 16) |
           ((uint32_t)path << 22) | ((uint32_t)magnified << 25) | ((uint32_t)(a < 32) << 26);

    for (int lane = 0; lane < 32; ++lane) {
        if (!inframe[lane]) continue;
        size_t pix = (size_t)py[lane] * F->Wf + px[lane];
        for (int ch = 0; ch < 4; ++ch) F->out[4 * pix + ch] = col[lane][ch];
        if (F->produced_id) F->produced_id[pix] = prod[lane];
        if (F->selection) F->selection[pix] = sel[lane];
    }
}

/* ========================================================================= */
/* Bicubic filters: cubic B-spline and Catmull-Rom (§5.4; the      */
/* 4x4 footprint and "<= 2 evaluations per lane", Fig. 13          */
/* P:1731-1753).  Readings R-24 .. R-28 in DESIGN.md.                         */
/* ========================================================================= */
enum { FILTER_BILINEAR = 0, FILTER_BSPLINE = 1, FILTER_CATMULL_ROM = 2 };

/* R-25: weights of the taps x0-1, x0, x0+1, x0+2 at fraction s in [0,1); the
 * uniform cubic B-spline and Catmull-Rom kernels (the paper names the filters,
 * P:704-708, not their formulas).  fp32, one rounding per operation, in the
 * order written (they decide integers: STF / C+ picks). */
void oracle_cubic_weights(int filter, float s, float w[4])
{
    float r = 1.0f - s;
    float s2 = s * s, s3 = s2 * s, r2 = r * r;
    if (filter == FILTER_BSPLINE) {
        float r3 = r2 * r;
        w[0] = r3 / 6.0f;
        w[1] = ((3.0f * s3 - 6.0f * s2) + 4.0f) / 6.0f;
        w[2] = (((3.0f * s2 - 3.0f * s3) + 3.0f * s) + 1.0f) / 6.0f;
        w[3] = s3 / 6.0f;
    } else {
        w[0] = -0.5f * (s * r2);
        w[1] = ((3.0f * s3 - 5.0f * s2) + 2.0f) * 0.5f;
        w[2] = ((4.0f * s2 - 3.0f * s3) + s) * 0.5f;
        w[3] = -0.5f * (s2 * r);
    }
}

typedef struct {
    int active, magnified;
    int x[4], y[4];        /* clamped tap columns x0-1+i and rows y0-1+j (R-24)          */
    float wx[4], wy[4];    /* tap weights (R-25)                                           */
    int xa, nc, ya, nr;    /* distinct columns xa..xa+nc-1, rows ya..ya+nr-1              */
    float mx[4], my[4];    /* per distinct column / row: sum of its taps' weights, fp32,
                              taps in ascending order (clamp duplicates merge, R-25)        */
} lane16_t;

static void make_lane16(lane16_t *L, int filter, const float *uv, const uint16_t *grad, int W, int H)
{
    /* R-24: the same coordinate rule as the bilinear footprint (R-2) */
    float uc = fminf(fmaxf(uv[0], 0.0f), 1.0f);
    float vc = fminf(fmaxf(uv[1], 0.0f), 1.0f);
    float fx = fmaf(uc, (float)W, -0.5f), fy = fmaf(vc, (float)H, -0.5f);
    float flx = floorf(fx), fly = floorf(fy);
    int x0 = (int)flx, y0 = (int)fly;
    oracle_cubic_weights(filter, fx - flx, L->wx);
    oracle_cubic_weights(filter, fy - fly, L->wy);
    for (int i = 0; i < 4; ++i) {
        L->x[i] = clampi(x0 - 1 + i, 0, W - 1);
        L->y[i] = clampi(y0 - 1 + i, 0, H - 1);
    }
    L->xa = L->x[0]; L->nc = L->x[3] - L->x[0] + 1;
    L->ya = L->y[0]; L->nr = L->y[3] - L->y[0] + 1;
    for (int i = 0; i < 4; ++i) { L->mx[i] = 0.0f; L->my[i] = 0.0f; }
    for (int i = 0; i < 4; ++i) {
        L->mx[L->x[i] - L->xa] = L->mx[L->x[i] - L->xa] + L->wx[i];
        L->my[L->y[i] - L->ya] = L->my[L->y[i] - L->ya] + L->wy[i];
    }
    L->magnified = 0;
    if (grad) {   /* R-20, unchanged */
        float g0 = half_to_float(grad[0]), g1 = half_to_float(grad[1]);
        float g2 = half_to_float(grad[2]), g3 = half_to_float(grad[3]);
        volatile float a0 = g0 * g0, a1 = g1 * g1, a2 = g2 * g2, a3 = g3 * g3;
        float rx = a0 + a1, ry = a2 + a3;
        L->magnified = ((rx > ry ? rx : ry) <= 1.0f);
    }
}

static uint32_t cell_id(const lane16_t *L, int c, int r, int W)
{
    return (uint32_t)(L->ya + r) * (uint32_t)W + (uint32_t)(L->xa + c);
}

/* the plain definition: sum over the 16 taps of wx_i * wy_j * p(x_i, y_j), fp64 */
static void blend16_exact(const tex_t *tex, const lane16_t *L, double c[4])
{
    for (int ch = 0; ch < 4; ++ch) c[ch] = 0.0;
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) {
            double p[4];
            produce(tex, (uint32_t)L->y[j] * (uint32_t)tex->W + (uint32_t)L->x[i], p);
            double w = (double)L->wx[i] * (double)L->wy[j];
            for (int ch = 0; ch < 4; ++ch) c[ch] += w * p[ch];
        }
}

/* R-26 one-tap STF for a separable filter: column ~ |wx|, row ~ |wy| (so P(tap) =
 * |w_ij| / sum |w|, "absolute values of filter weights"), each by the
 * inverse CDF in fp32 (first cumulative sum > u * S, else the last nonzero tap). */
static int cubic_pick(const float w[4], float u, float *S_out)
{
    float S = 0.0f;
    int last = 0;
    for (int i = 0; i < 4; ++i) { S = S + fabsf(w[i]); if (w[i] != 0.0f) last = i; }
    volatile float target = u * S;
    float cum = 0.0f;
    *S_out = S;
    for (int i = 0; i < 4; ++i) {
        cum = cum + fabsf(w[i]);
        if (cum > target) return i;
    }
    return last;
}

/* the one-tap estimate sign(w) * (Sx * Sy) * p of lane L's STF tap; returns its id */
static uint32_t stf16(const tex_t *tex, const lane16_t *L, const double u[4], double c[4])
{
    float Sx, Sy;
    int i = cubic_pick(L->wx, (float)u[0], &Sx);
    int j = cubic_pick(L->wy, (float)u[1], &Sy);
    uint32_t id = (uint32_t)L->y[j] * (uint32_t)tex->W + (uint32_t)L->x[i];
    if (c) {
        double p[4];
        produce(tex, id, p);
        double sgn = ((L->wx[i] < 0.0f) != (L->wy[j] < 0.0f)) ? -1.0 : 1.0;
        for (int ch = 0; ch < 4; ++ch) c[ch] = sgn * (double)Sx * (double)Sy * p[ch];
    }
    return id;
}

/* R-27 positivized STF (the paper's 2-evaluation baseline for filters with negative
 * lobes): taps k = 4j + i in row-major order with w_k = wx_i * wy_j (fp32);
 * W+ = sum of positive w_k, W- = sum of -w_k over negative ones (fp32, k ascending);
 * p+ ~ w_k over the positive taps (u0), p- ~ -w_k over the negative taps (u1), by the
 * inverse CDF as in R-26; c = W+ p+ - W- p-.  Returns the number of evaluations. */
static int stf16_positivized(const tex_t *tex, const lane16_t *L, const double u[4], double c[4])
{
    float wk[16], Wp = 0.0f, Wn = 0.0f;
    int lastp = -1, lastn = -1;
    for (int k = 0; k < 16; ++k) {
        wk[k] = L->wx[k & 3] * L->wy[k >> 2];
        if (wk[k] > 0.0f) { Wp = Wp + wk[k]; lastp = k; }
        else if (wk[k] < 0.0f) { Wn = Wn + (-wk[k]); lastn = k; }
    }
    for (int ch = 0; ch < 4; ++ch) c[ch] = 0.0;
    int evals = 0;
    for (int lobe = 0; lobe < 2; ++lobe) {
        float Wl = lobe ? Wn : Wp;
        if (!(Wl > 0.0f)) continue;
        volatile float target = (float)u[lobe] * Wl;
        float cum = 0.0f;
        int pick = lobe ? lastn : lastp;
        for (int k = 0; k < 16; ++k) {
            if (lobe ? !(wk[k] < 0.0f) : !(wk[k] > 0.0f)) continue;
            cum = cum + (lobe ? -wk[k] : wk[k]);
            if (cum > target) { pick = k; break; }
        }
        double p[4];
        produce(tex, (uint32_t)L->y[pick >> 2] * (uint32_t)tex->W + (uint32_t)L->x[pick & 3], p);
        for (int ch = 0; ch < 4; ++ch) c[ch] += (lobe ? -(double)Wl : (double)Wl) * p[ch];
        ++evals;
    }
    return evals;
}

/* Eq. 1 over the known cells of L's footprint: distinct texels in
 * row-major order with merged weight mw = mx[c] * my[r] (fp32) != 0 (R-14, R-28). */
static void blend16_fallback(const tex_t *tex, const lane16_t *L, const uint32_t *produced, int nprod,
                             double c[4])
{
    int all_known = 1, N = 0;
    double Swp[4] = { 0, 0, 0, 0 }, Sp[4] = { 0, 0, 0, 0 }, Sw = 0.0, plast[4] = { 0, 0, 0, 0 };
    for (int r = 0; r < L->nr; ++r)
        for (int q = 0; q < L->nc; ++q) {
            float mw = L->mx[q] * L->my[r];
            if (mw == 0.0f) continue;
            uint32_t id = cell_id(L, q, r, tex->W);
            if (!in_list(produced, nprod, id)) { all_known = 0; continue; }
            double p[4];
            produce(tex, id, p);
            for (int ch = 0; ch < 4; ++ch) { Swp[ch] += (double)mw * p[ch]; Sp[ch] += p[ch]; plast[ch] = p[ch]; }
            Sw += (double)mw;
            ++N;
        }
    if (all_known) { blend16_exact(tex, L, c); return; }
    if (N == 1) { for (int ch = 0; ch < 4; ++ch) c[ch] = plast[ch]; return; }
    for (int ch = 0; ch < 4; ++ch) c[ch] = Swp[ch] + (1.0 - Sw) * Sp[ch] / N;   /* Eq. 1 */
}

static void wave_bicubic(const frame_t *F, int filter, int E, int wx, int wy)
{
    const tex_t *tex = F->tex;
    const int W = tex->W;
    lane16_t L[32];
    int px[32], py[32], inframe[32];
    uint32_t A = 0;
    for (int lane = 0; lane < 32; ++lane) {
        px[lane] = wx * 8 + (lane & 7);
        py[lane] = wy * 4 + (lane >> 3);
        inframe[lane] = px[lane] < F->Wf && py[lane] < F->Hf;
        memset(&L[lane], 0, sizeof(lane16_t));
        if (!inframe[lane]) continue;
        size_t pix = (size_t)py[lane] * F->Wf + px[lane];
        const float *uvp = F->uv + 2 * pix;
        if (isnan(uvp[0])) continue;
        L[lane].active = 1;
        A |= 1u << lane;
        make_lane16(&L[lane], filter, uvp, F->grad ? F->grad + 4 * pix : NULL, W, tex->H);
    }
    int a = __builtin_popcount(A);
    int nwx = (F->Wf + 7) / 8;
    uint32_t *rec = &F->rec[(size_t)wy * nwx + wx];
    double col[32][4];
    for (int lane = 0; lane < 32; ++lane) for (int ch = 0; ch < 4; ++ch) col[lane][ch] = 0.0;
    /* debug outputs of the one-evaluation paths (fallbacks): the texel a lane produced and the
     * C+ spare-lane fields, as in the bilinear wave(); the exact path (up to E evaluations per
     * lane) and the full / positivized filters report none */
    uint32_t prod[32], sel[32];
    for (int lane = 0; lane < 32; ++lane) { prod[lane] = INVALID_ID; sel[lane] = 0; }
    int magnified = 0;
    if (F->grad && a > 0) {
        magnified = 1;
        for (int lane = 0; lane < 32; ++lane) if (L[lane].active && !L[lane].magnified) magnified = 0;
    }
    int act[32];
    for (int r = 0; r < a; ++r) act[r] = oracle_h((uint32_t)r, A);
    double u[32][4];
    for (int lane = 0; lane < 32; ++lane)
        if (L[lane].active) pixel_uniforms(px[lane], py[lane], F->frame, F->seed, u[lane]);

    int n = 0xFF, evals = 0, path = 0, run_fallback = -1;
    if (F->mode == M_4TAP) {
        /* the full filter: 16 evaluations per pixel */
        path = PATH_4TAP;
        for (int lane = 0; lane < 32; ++lane) if (L[lane].active) blend16_exact(tex, &L[lane], col[lane]);
        evals = 16 * a;
    } else if (F->mode == M_STF) {
        path = PATH_STF;
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) evals += stf16_positivized(tex, &L[lane], u[lane], col[lane]);
    } else {
        /* collect: the exact set of distinct texels over all active 4x4 footprints (R-4) */
        uint32_t *U = (uint32_t *)malloc(sizeof(uint32_t) * 512);
        int m = 0, minx = 1 << 30, maxx = -1, miny = 1 << 30, maxy = -1;
        for (int lane = 0; lane < 32; ++lane) {
            if (!L[lane].active) continue;
            for (int r = 0; r < L[lane].nr; ++r)
                for (int q = 0; q < L[lane].nc; ++q) U[m++] = cell_id(&L[lane], q, r, W);
            if (L[lane].xa < minx) minx = L[lane].xa;
            if (L[lane].ya < miny) miny = L[lane].ya;
            if (L[lane].xa + L[lane].nc - 1 > maxx) maxx = L[lane].xa + L[lane].nc - 1;
            if (L[lane].ya + L[lane].nr - 1 > maxy) maxy = L[lane].ya + L[lane].nr - 1;
        }
        int nu = sort_unique(U, m);
        free(U);
        const int cap = E * a;                      /* <= E evaluations per lane */
        n = nu < cap + 1 ? nu : cap + 1;            /* record: n saturated at E*a + 1 (R-28) */
        int ok = 0, bw = 0, bh = 0;
        if (a > 0) {
            bw = maxx - minx + 1;
            bh = maxy - miny + 1;
            if (F->mode == M_BOX) ok = bw * bh <= cap;
            else if (F->mode == M_MASK16) ok = bw <= 16 && bh <= 16 && nu <= cap;
            else if (F->mode == M_MASK11) ok = bw <= 11 && bh <= 11 && nu <= cap;
            else ok = nu <= cap;
        }
        if (a > 0 && ok && !(F->flags & FL_FORCE_FALLBACK)) {
            /* rank r (or Box index r) is produced by lane h(r mod a, A) as its
             * (r div a)-th evaluation; the result is the plain 16-tap filter */
            path = PATH_EXACT;
            evals = (F->mode == M_BOX) ? bw * bh : nu;
            for (int lane = 0; lane < 32; ++lane) if (L[lane].active) blend16_exact(tex, &L[lane], col[lane]);
        } else {
            run_fallback = F->fallback;
            path = PATH_FB_STF + F->fallback;
        }
    }

    if (run_fallback == FB_STF) {
        for (int lane = 0; lane < 32; ++lane) if (L[lane].active) prod[lane] = stf16(tex, &L[lane], u[lane], col[lane]);
        evals = a;
    } else if (run_fallback == FB_C || run_fallback == FB_CPLUS) {
        /* planned texels: every lane's one-tap STF choice (R-26) */
        uint32_t P[32], produced[32];
        int np = 0, nprod = 0;
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) P[np++] = stf16(tex, &L[lane], u[lane], NULL);
        if (run_fallback == FB_C) {
            for (int i = 0; i < np; ++i) { produced[nprod++] = P[i]; prod[act[i]] = P[i]; }   /* every lane produces */
            evals = a;
        } else {
            np = sort_unique(P, np);                                     /* C+ plan (R-17) */
            for (int i = 0; i < np; ++i) { produced[nprod++] = P[i]; prod[act[i]] = P[i]; }
            for (int j = np; j < a; ++j) {                               /* Eq. 2 spare lanes */
                int cl = act[j];
                const int sl = act[oracle_eq2(j, np, a)];
                sel[cl] |= (1u << 5) | ((uint32_t)sl << 8);
                const lane16_t *Ll = &L[sl];
                uint32_t fid[16]; float fw[16]; int nf = 0;
                for (int r = 0; r < Ll->nr; ++r)
                    for (int q = 0; q < Ll->nc; ++q) {
                        float mw = Ll->mx[q] * Ll->my[r];
                        uint32_t id = cell_id(Ll, q, r, W);
                        if (mw == 0.0f || in_list(P, np, id)) continue;
                        fid[nf] = id; fw[nf] = fabsf(mw); ++nf;
                    }
                if (nf == 0) continue;
                float wsum = 0.0f;
                for (int q = 0; q < nf; ++q) wsum = wsum + fw[q];
                volatile float target = (float)u[cl][2] * wsum;
                int pick = nf - 1;
                float cum = 0.0f;
                for (int q = 0; q < nf; ++q) {
                    cum = cum + fw[q];
                    if (cum > target) { pick = q; break; }
                }
                produced[nprod++] = fid[pick];
                prod[cl] = fid[pick];
                sel[cl] |= 1u << 4;
            }
            evals = nprod;
        }
        for (int lane = 0; lane < 32; ++lane)
            if (L[lane].active) blend16_fallback(tex, &L[lane], produced, nprod, col[lane]);
    }

    if (a == 0) { evals = 0; path = 0; if (F->mode >= M_COLLAB) n = 0; }
    *rec = (uint32_t)(evals & 0xFF) | ((uint32_t)(n & 0xFF) << 8) | ((uint32_t)a << 16) |
           ((uint32_t)path << 22) | ((uint32_t)magnified << 25) | ((uint32_t)(a < 32) << 26) |
           ((uint32_t)((evals >> 8) & 7) << 27);
    for (int lane = 0; lane < 32; ++lane) {
        if (!inframe[lane]) continue;
        size_t pix = (size_t)py[lane] * F->Wf + px[lane];
        for (int ch = 0; ch < 4; ++ch) F->out[4 * pix + ch] = col[lane][ch];
        if (F->produced_id) F->produced_id[pix] = prod[lane];
        if (F->selection) F->selection[pix] = sel[lane];
    }
}

/* ------------------------------------------------------------------------- */
/* Frame entry.  Returns 0, or -1 on invalid arguments.                       */
/*   out: fp64 [Hf][Wf][4]; rec: u32 [ceil(Hf/4)][ceil(Wf/8)];                */
/*   produced_id / selection: u32 [Hf][Wf] or NULL.                           */
/* ------------------------------------------------------------------------- */
static int check_args(int format, int W, int H, const uint8_t *bc1, const uint16_t *latent, const float *mlp,
                      const float *uv, int Wf, int Hf, int mode, int fallback, int filter, int max_evals,
                      const double *out, const uint32_t *rec)
{
    if (W <= 0 || H <= 0 || Wf <= 0 || Hf <= 0 || !uv || !out || !rec) return -1;
    if (format == FMT_BC1 && (!bc1 || W % 4 || H % 4)) return -1;
    if (format == FMT_LATENT_MLP && (!latent || !mlp || W % 4 || H % 4)) return -1;
    if (format != FMT_BC1 && format != FMT_LATENT_MLP) return -1;
    if (mode < 0 || mode > 6 || fallback < 0 || fallback > 3) return -1;
    if (filter < FILTER_BILINEAR || filter > FILTER_CATMULL_ROM || max_evals < 0 || max_evals > 2) return -1;
    if (filter == FILTER_BILINEAR && max_evals > 1) return -1;
    if (filter != FILTER_BILINEAR && (mode == M_WC || fallback == FB_WC)) return -1;   /* R-28 */
    return 0;
}

static void run_wave(const frame_t *F, int filter, int E, int wx, int wy)
{
    if (filter == FILTER_BILINEAR) wave(F, wx, wy);
    else wave_bicubic(F, filter, E, wx, wy);
}

/* filter: 0 bilinear, 1 cubic B-spline, 2 Catmull-Rom (R-25); max_evals: texel
 * evaluations per lane on the exact path, 0/1 or 2 (bicubic only). */
int oracle_filter_frame2(int format, int W, int H, const uint8_t *bc1, const uint16_t *latent,
                         const float *mlp, const float *uv, const uint16_t *grad, int Wf, int Hf,
                         int mode, int fallback, unsigned flags, uint64_t seed, uint32_t frame_index,
                         int filter, int max_evals,
                         double *out, uint32_t *rec, uint32_t *produced_id, uint32_t *selection)
{
    if (check_args(format, W, H, bc1, latent, mlp, uv, Wf, Hf, mode, fallback, filter, max_evals, out, rec))
        return -1;
    tex_t tex = { format, W, H, bc1, latent, mlp };
    frame_t F = { &tex, uv, grad, Wf, Hf, mode, fallback, flags, seed, frame_index,
                  out, rec, produced_id, selection };
    int E = max_evals < 1 ? 1 : max_evals;
    int nwx = (Wf + 7) / 8, nwy = (Hf + 3) / 4;
    long nw = (long)nwx * nwy;
#pragma omp parallel for schedule(dynamic, 64)
    for (long w = 0; w < nw; ++w) run_wave(&F, filter, E, (int)(w % nwx), (int)(w / nwx));
    return 0;
}

int oracle_filter_frame(int format, int W, int H, const uint8_t *bc1, const uint16_t *latent,
                        const float *mlp, const float *uv, const uint16_t *grad, int Wf, int Hf,
                        int mode, int fallback, unsigned flags, uint64_t seed, uint32_t frame_index,
                        double *out, uint32_t *rec, uint32_t *produced_id, uint32_t *selection)
{
    return oracle_filter_frame2(format, W, H, bc1, latent, mlp, uv, grad, Wf, Hf, mode, fallback, flags, seed,
                                frame_index, FILTER_BILINEAR, 1, out, rec, produced_id, selection);
}

/* Same, restricted to a list of waves (sampled parity at full size). */
int oracle_filter_waves2(int format, int W, int H, const uint8_t *bc1, const uint16_t *latent,
                         const float *mlp, const float *uv, const uint16_t *grad, int Wf, int Hf,
                         int mode, int fallback, unsigned flags, uint64_t seed, uint32_t frame_index,
                         int filter, int max_evals, const int32_t *wave_list, int nlist,
                         double *out, uint32_t *rec, uint32_t *produced_id, uint32_t *selection)
{
    if (!wave_list ||
        check_args(format, W, H, bc1, latent, mlp, uv, Wf, Hf, mode, fallback, filter, max_evals, out, rec))
        return -1;
    tex_t tex = { format, W, H, bc1, latent, mlp };
    frame_t F = { &tex, uv, grad, Wf, Hf, mode, fallback, flags, seed, frame_index,
                  out, rec, produced_id, selection };
    int E = max_evals < 1 ? 1 : max_evals;
    int nwx = (Wf + 7) / 8;
#pragma omp parallel for schedule(dynamic, 16)
    for (int i = 0; i < nlist; ++i) run_wave(&F, filter, E, wave_list[i] % nwx, wave_list[i] / nwx);
    return 0;
}

int oracle_filter_waves(int format, int W, int H, const uint8_t *bc1, const uint16_t *latent,
                        const float *mlp, const float *uv, const uint16_t *grad, int Wf, int Hf,
                        int mode, int fallback, unsigned flags, uint64_t seed, uint32_t frame_index,
                        const int32_t *wave_list, int nlist,
                        double *out, uint32_t *rec, uint32_t *produced_id, uint32_t *selection)
{
    return oracle_filter_waves2(format, W, H, bc1, latent, mlp, uv, grad, Wf, Hf, mode, fallback, flags, seed,
                                frame_index, FILTER_BILINEAR, 1, wave_list, nlist, out, rec, produced_id,
                                selection);
}

/* Thread count of the OpenMP loops over waves (bench.py's single-thread timing); returns the
 * previous maximum.  Scheduling only: results do not depend on it. */
#ifdef _OPENMP
#include <omp.h>
#endif
int oracle_set_threads(int n)
{
#ifdef _OPENMP
    int prev = omp_get_max_threads();
    if (n > 0) omp_set_num_threads(n);
    return prev;
#else
    (void)n;
    return 1;
#endif
}

/* Number of distinct texels in an arbitrary list (brute force, for pins). */
int oracle_unique_count(const uint32_t *ids, int n)
{
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    memcpy(tmp, ids, sizeof(uint32_t) * (size_t)n);
    int m = sort_unique(tmp, n);
    free(tmp);
    return m;
}
