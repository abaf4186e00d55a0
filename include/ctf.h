/*
 * ctf.h — C ABI of the B200 collaborative texture filtering hot path.
 *
 * Method: "Collaborative Texture Filtering", arXiv 2506.17770 (PAPER.md; P:n
 * below is a PAPER.md line).  One 8x4-pixel wave is one 32-lane warp
 * (P:266-268).  Each lane forms its bilinear 2x2 footprint; the
 * warp collects the unique texels it needs (step 1), each lane
 * produces at most one texel (step 2), and each lane gathers its
 * texels from the other lanes and filters them (step 3), which equals
 * plain bilinear filtering with zero error whenever the wave needs no more
 * unique texels than it has active lanes (edge
 * remapping, suppl. §2).  Otherwise a fallback runs: one-tap STF
 * (P:136-141), a wave-communication STF stand-in, or the paper's
 * C (Eq. 1) and C+ (Eq. 2) estimators.
 *
 * Conventions (all entry points):
 *  - Every pointer named *_dev is a DEVICE pointer owned by the caller; *_host
 *    pointers are host memory owned by the caller (pinned for overlap).  The
 *    library never allocates on the filtering path and keeps no global state:
 *    calls are re-entrant across streams and devices (the current device is
 *    the caller's).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device work is enqueued asynchronously on it unless stated otherwise.
 *  - Return value: CTF_OK or a negative ctf_status, decided synchronously by
 *    host-side validation before anything is enqueued (CTF_ECUDA reports a
 *    launch error; execution faults surface at the caller's next sync).
 *  - Layouts are row-major; no padding between rows or frames.
 *
 * Wave / pixel layout: wave (wx, wy) covers pixels x in [8wx, 8wx+8),
 * y in [4wy, 4wy+4); lane = 8*(y & 3) + (x & 7) (row-major; R-1).
 * A lane is ACTIVE iff its pixel is inside the frame and u is not NaN.
 */
#ifndef CTF_H_
#define CTF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTF_ABI_VERSION 6

typedef enum {
    CTF_OK = 0,
    CTF_EINVAL = -1,       /* null required pointer, bad size, unknown enum value          */
    CTF_EUNSUPPORTED = -2, /* valid but not supported (e.g. W*H > 2^24 texels)              */
    CTF_EALIGN = -3,       /* uv not 8-byte aligned, out not 16-byte aligned, ...          */
    CTF_ECUDA = -4         /* a CUDA runtime call or kernel launch failed                   */
} ctf_status;

/* Texture formats: the texel "producer" of step 2. */
typedef enum {
    CTF_FMT_BC1 = 1,        /* synthetic BC1-style blocks (R-9)                  */
    CTF_FMT_LATENT_MLP = 2  /* NTC-style latent grid + MLP 12->32->32->4 (R-10) */
} ctf_format;

typedef enum { CTF_ADDR_CLAMP = 0 } ctf_addr;  /* clamp-to-edge (R-2 i; P:1050 omits it) */

typedef struct {
    int32_t format;          /* ctf_format                                                  */
    int32_t width, height;   /* texels; multiples of 4; width*height <= 2^24               */
    int32_t addr;            /* ctf_addr; must be CTF_ADDR_CLAMP                            */
    const void *data_dev;    /* BC1: 8-byte blocks [(H/4)][(W/4)]: u16 c0, u16 c1 (RGB565),
                                u32 2-bit codes, texel (x&3,y&3) at bit 2*(4*(y&3)+(x&3)).
                                LATENT_MLP: fp16 latents [(H/4)][(W/4)][8].                 */
    const float *mlp_dev;    /* LATENT_MLP: 1604 fp32 = W1[32][12] b1[32] W2[32][32] b2[32]
                                W3[4][32] b3[4]; NULL for BC1.                               */
    const float *mlp_host;   /* LATENT_MLP, REQUIRED (ABI 6): HOST copy of the same 1604
                                weights.  The kernels receive the weights by value in their
                                parameter block (constant bank), so a launch reads them from
                                here and never copies from the device (no hidden
                                synchronisation; calls stay asynchronous and capturable in a
                                CUDA graph).  NULL with LATENT_MLP -> CTF_EINVAL.  NULL for BC1. */
} ctf_texture;

/* Filter modes (P:606-609 naming: method + fallback in parentheses). */
typedef enum {
    CTF_MODE_BILINEAR_4TAP = 0, /* classic bilinear, 4 evaluations per pixel      */
    CTF_MODE_STF = 1,           /* one-tap stochastic texture filtering (Pharr 2024) */
    CTF_MODE_WAVECOMM = 2,      /* wave-communication STF stand-in (R-16)        */
    CTF_MODE_COLLAB = 3,        /* collaborative filtering, List semantics: exact iff the
                                   wave's unique texels n <= active lanes (§3.1)  */
    CTF_MODE_BOX = 4,           /* Box Sampling: exact iff AABB area <= active lanes; lanes
                                   produce the whole AABB (§3.2)    */
    CTF_MODE_MASK16 = 5,        /* Mask Sampling 16x16: exact iff AABB <= 16x16 and n <= a
                                   (§3.3)                            */
    CTF_MODE_MASK11 = 6         /* Mask Sampling 11x11                           */
} ctf_mode;

typedef enum {
    CTF_FB_STF = 0,      /* one-tap STF                                                    */
    CTF_FB_WAVECOMM = 1, /* WC stand-in                                                    */
    CTF_FB_C = 2,        /* "C": Eq. 1 over the wave's produced STF texels     */
    CTF_FB_CPLUS = 3     /* "C+": deduplicated plan + Eq. 2 spare lanes + Eq. 1 */
} ctf_fallback;

enum {
    CTF_FLAG_DEBUG = 1u << 0,          /* fill the ctf_debug buffers                        */
    CTF_FLAG_FORCE_FALLBACK = 1u << 1, /* COLLAB: every wave runs the fallback */
    CTF_FLAG_SEPARATE_PASSES = 1u << 2 /* (ABI 6) BC1 collaborative bilinear: always run the
                                          multi-kernel pipeline (lean exact kernel, then the
                                          waves it leaves in their own passes), never the
                                          single fused launch the library picks for calls of
                                          at most 131072 waves.  Results are identical.     */
};

/* Texture filters (§5.4 "Bicubic Filtering").  The bicubic filters use a 4x4
 * footprint (taps x0-1..x0+2, y0-1..y0+2, clamp-to-edge) with the weights of DESIGN.md
 * R-25; every mode above applies except WAVECOMM (mode and fallback -> EUNSUPPORTED), and
 * with a bicubic filter:
 *   - BILINEAR_4TAP means the full filter (16 evaluations per pixel);
 *   - STF is the positivized two-lobe estimator, 1-2 evaluations per pixel;
 *   - the fallbacks draw their one-tap samples with probability |w| / sum |w|;
 *   - max_evals = 2 lets the exact path use up to 2 evaluations per lane (n <= 2a,
 *     P:917-931 and Fig. 13b); the fallbacks keep <= 1. */
typedef enum {
    CTF_FILTER_BILINEAR = 0,
    CTF_FILTER_BSPLINE = 1,      /* uniform cubic B-spline (approximating, weights >= 0)      */
    CTF_FILTER_CATMULL_ROM = 2   /* Catmull-Rom (interpolating, negative lobes)               */
} ctf_filter;

typedef struct {
    int32_t mode;          /* ctf_mode                                                     */
    int32_t fallback;      /* ctf_fallback; used by the collaborative modes (COLLAB..MASK11)*/
    uint32_t flags;        /* CTF_FLAG_*                                                   */
    uint32_t frame_index;  /* RNG counter word; batch frame f uses frame_index + f          */
    uint64_t seed;         /* RNG key (R-11: Philox4x32-10, ctr = (x, y, frame, 0))         */
    int32_t filter;        /* ctf_filter (ABI 2); 0 = bilinear                             */
    int32_t max_evals;     /* exact-path evaluations per lane: 0 or 1, or 2 (bicubic only)  */
    void *workspace_dev;   /* optional device scratch (ABI 4), >= ctf_filter_workspace_bytes()
                              bytes, 16-byte aligned, owned by the caller, contents need no
                              initialisation; used by the COLLAB / BOX / MASK16 / MASK11 bilinear paths for
                              compact work lists of its fallback / general waves (no record
                              scans, balanced second passes).  NULL: the record buffer doubles
                              as the work list.  Results are identical either way.  Calls
                              that share a workspace must be ordered (same stream).        */
    uint64_t workspace_bytes;
    int32_t row0;          /* (ABI 6) frame row of the first buffer row, a multiple of 4, >= 0:
                              the buffers hold rows [row0, row0 + Hf) of a taller frame (strip
                              sharding).  Only the RNG counter uses the frame row
                              (ctr = (x, row0 + y, frame, 0)); waves never read outside their
                              8x4 pixels, so a strip's results equal the same rows
                              of the whole frame bit for bit.  0 for whole frames.          */
    int32_t reserved_;     /* must be 0                                                     */
} ctf_params;

/* Optional per-pixel debug outputs (only with CTF_FLAG_DEBUG; any may be NULL). */
typedef struct {
    uint32_t *produced_id_dev; /* [frames][Hf][Wf]: texel id (y*W+x) this lane produced,
                                  0xFFFFFFFF = none (and for 4TAP)                          */
    uint32_t *selection_dev;   /* [frames][Hf][Wf]: b0-1 STF corner (UL,UR,LL,LR); b2-3 C+
                                  extra corner; b4 has-extra; b5 spare lane; b8-12 served
                                  lane l (Eq. 2)                                             */
    uint32_t *unread_dev;      /* [1], accumulated: exact-path gathers from lanes that did
                                  not produce (must stay 0)                           */
} ctf_debug;

/*
 * Per-wave record (u32), one per wave, [frames][ceil(Hf/4)][ceil(Wf/8)]:
 *   bits 0-7   texel evaluations in the wave, low 8 bits (exact: n, Box: AABB area;
 *              4TAP: 4a (16a bicubic); STF/WC/C: a (positivized STF: 1-2 per lane); C+:
 *              n_p + spare lanes that produced); bits 27-29 hold bits 8-10
 *   bits 8-15  n = number of unique texels the wave needs (collaborative modes; 0xFF
 *              for 4TAP / STF / WC).  Bicubic: saturated at max_evals * a + 1 (R-28)
 *   bits 16-21 a = active lanes
 *   bits 22-24 path: 0 exact, 1 fb-STF, 2 fb-WC, 3 fb-C, 4 fb-C+, 5 4TAP, 6 STF, 7 WC
 *   bit  25    magnified: grad given and every active lane has
 *              max(|J_x|^2, |J_y|^2) <= 1 in texel units (R-20)
 *   bit  26    partial: a < 32
 *   bits 27-29 evals bits 8-10
 */
#define CTF_REC_EVALS(r) (((r) & 0xFFu) | ((((r) >> 27) & 0x7u) << 8))
#define CTF_REC_N(r) (((r) >> 8) & 0xFFu)
#define CTF_REC_A(r) (((r) >> 16) & 0x3Fu)
#define CTF_REC_PATH(r) (((r) >> 22) & 0x7u)
#define CTF_REC_MAGNIFIED(r) (((r) >> 25) & 1u)
#define CTF_REC_PARTIAL(r) (((r) >> 26) & 1u)

/*
 * Filter one frame.
 *   tex        texture descriptor (host struct; its pointers are device pointers)
 *   uv_dev     float[Hf][Wf][2] normalised (u, v); u = NaN marks an uncovered pixel.
 *              Coordinates are clamped to [0, 1] before use (clamp-to-edge, R-2).  8-B aligned.
 *   grad_dev   fp16 bits [Hf][Wf][4] = (du/dx, dv/dx, du/dy, dv/dy) in texel units, or
 *              NULL (then the magnified bit is 0).  8-B aligned.
 *   Wf, Hf     frame size in pixels, any value >= 1 (partial waves at the right/bottom).
 *   p          parameters (host struct).
 *   out_dev    float[Hf][Wf][4] RGBA; uncovered pixels get (0,0,0,0).  16-B aligned.
 *   rec_dev    u32 per-wave records (layout above).
 *   dbg        NULL or debug buffers (used only with CTF_FLAG_DEBUG).
 */
int ctf_filter_frame(const ctf_texture *tex, const float *uv_dev, const uint16_t *grad_dev,
                     int32_t Wf, int32_t Hf, const ctf_params *p, float *out_dev,
                     uint32_t *rec_dev, const ctf_debug *dbg, void *stream);

/*
 * Filter `frames` consecutive frames in one pass over all waves (one kernel per path step;
 * ctf_launches_per_call counts them).  uv_dev/grad_dev/out_dev/rec_dev (and debug buffers)
 * hold `frames` frames back to back; frame f is filtered with frame_index =
 * p->frame_index + f.  Same results as `frames` calls of ctf_filter_frame.
 * All work is enqueued on `stream` (no library-owned streams, events or allocations).
 */
int ctf_filter_batch(const ctf_texture *tex, const float *uv_dev, const uint16_t *grad_dev,
                     int32_t Wf, int32_t Hf, int32_t frames, const ctf_params *p,
                     float *out_dev, uint32_t *rec_dev, const ctf_debug *dbg, void *stream);

/* Frame / batch totals (PSNR per P:1449-1469). */
typedef struct {
    uint64_t waves_live, waves_partial, waves_exact, waves_fallback, waves_magnified;
    uint64_t pixels_active, pixels_in_magnified_waves, texel_evals, texel_evals_in_magnified_waves;
    uint32_t max_evals_per_lane, max_unique_per_wave;
    uint64_t unique_hist[129];      /* live COLLAB waves by n (0..128)                      */
    double sum_sq_err;              /* Sum over pixels and 4 channels of (out - ref)^2      */
    float max_abs_err;              /* max |out - ref| over pixels and channels             */
    uint32_t pad_;
    uint64_t err_pixels;            /* pixels compared (all in-frame pixels of the batch)   */
} ctf_frame_stats;

/*
 * Reduce per-wave records (and optionally the error of out vs ref) of `frames` frames
 * into *host_out.  out_dev/ref_dev may both be NULL (no error terms) or both non-NULL
 * (float[frames][Hf][Wf][4]).  Deterministic (fixed reduction order).  Allocates a small
 * stream-ordered scratch buffer and SYNCHRONISES `stream` before returning.
 */
int ctf_stats(const uint32_t *rec_dev, int32_t Wf, int32_t Hf, int32_t frames,
              const float *out_dev, const float *ref_dev, ctf_frame_stats *host_out, void *stream);

/*
 * End-to-end entry with HOST buffers: copies uv/grad host->device, filters, and copies
 * out/records device->host, pipelined in chunks of `chunk_frames` frames over two
 * internal streams so copies overlap the kernel.  The texture must already be on the
 * device.  Device staging comes from the caller's workspace (size from
 * ctf_host_workspace_bytes).  Returns after everything has completed (synchronous).
 * grad_host may be NULL.  rec_host may be NULL (records not returned).
 */
size_t ctf_host_workspace_bytes(int32_t Wf, int32_t Hf, int32_t chunk_frames, int with_grad);
int ctf_filter_frames_host(const ctf_texture *tex, const float *uv_host, const uint16_t *grad_host,
                           int32_t Wf, int32_t Hf, int32_t frames, int32_t chunk_frames,
                           const ctf_params *p, float *out_host, uint32_t *rec_host,
                           void *workspace_dev, size_t workspace_bytes, void *stream);

/* Bytes of ctf_params.workspace_dev for `frames` frames of Wf x Hf (8 bytes per wave + 256). */
size_t ctf_filter_workspace_bytes(int32_t Wf, int32_t Hf, int32_t frames);

/*
 * Kernel launches one call above issues (for launch accounting): format / mode / filter as in
 * ctf_texture / ctf_params, a Wf x Hf frame, `frames` frames; flags: CTF_LAUNCH_BATCHED for
 * ctf_filter_batch (one pass over all frames) else ctf_filter_frame once per frame;
 * CTF_LAUNCH_SEPARATE_PASSES when ctf_params.flags has CTF_FLAG_SEPARATE_PASSES;
 * CTF_LAUNCH_WORKSPACE (a workspace in ctf_params) does not change the count.  The COLLAB /
 * BOX / MASK bilinear path is, for BC1, ONE fused kernel when a pass covers at most 131072
 * waves (and separate passes are not requested), else three (the lean exact kernel; then,
 * side by side, the third kernel over the waves it leaves with AABBs wider than 32x32 texels
 * — 64x64 bitmap windows, the sort-based general path beyond — and the wide-window kernel over
 * the others; plus an 8-byte cudaMemsetAsync of the work-list counters with a workspace, not
 * counted); two for the latent MLP (lean exact kernel + general path); every other path is
 * one.  Returns -1 for an invalid format / mode / filter / size.
 */
#define CTF_LAUNCH_BATCHED 1
#define CTF_LAUNCH_WORKSPACE 2
#define CTF_LAUNCH_SEPARATE_PASSES 4
int ctf_launches_per_call(int32_t format, int32_t mode, int32_t filter, int32_t Wf, int32_t Hf, int32_t frames,
                          int flags);
int ctf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CTF_H_ */
