// ctf_internal.h — launcher interface between the C-ABI shim and the kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace ctf {

constexpr int kMlpParams = 32 * 12 + 32 + 32 * 32 + 32 + 4 * 32 + 4;  // 1604 (R-10)

struct LaunchArgs {
    // texture
    int fmt, W, H;
    const void *tex_data;   // BC1 blocks or fp16 latents
    const float *mlp;       // device copy of the MLP weights
    const float *mlp_host;  // host copy (required; passed by value to the kernel)
    // frames
    const float *uv;        // [frames][Hf][Wf][2]
    const uint16_t *grad;   // [frames][Hf][Wf][4] fp16 bits or nullptr
    int Wf, Hf, frames;
    float *out;             // [frames][Hf][Wf][4]
    uint32_t *rec;          // [frames][nwy][nwx]
    // parameters
    int mode, fallback;
    uint32_t flags, frame_index;
    int row0;               // frame row of buffer row 0 (strip sharding; RNG counter only)
    uint64_t seed;
    int filter;             // ctf_filter: 0 bilinear, 1 B-spline, 2 Catmull-Rom
    int max_evals;          // exact-path evaluations per lane (1 or 2)
    // debug
    uint32_t *dbg_pid, *dbg_sel, *dbg_unread;
    // optional work lists (ctf_params.workspace_dev): [0] = #fallback waves, [1] = #general
    // waves, fallback list at [64], general list at [64 + waves]
    uint32_t *lists;
};

cudaError_t launch_filter_bc1(const LaunchArgs &a, cudaStream_t stream);  // ctf_filter.cu, CTF_TU_FMT=1
cudaError_t launch_filter_mlp(const LaunchArgs &a, cudaStream_t stream);  // ctf_filter.cu, CTF_TU_FMT=2
cudaError_t launch_bicubic_bc1(const LaunchArgs &a, cudaStream_t stream);  // ctf_bicubic.cu, CTF_TU_FMT=1
cudaError_t launch_bicubic_mlp(const LaunchArgs &a, cudaStream_t stream);  // ctf_bicubic.cu, CTF_TU_FMT=2
bool bicubic_built();
int launches_per_pass(int fmt, int mode, int filter, long long waves, unsigned flags);  // ctf_filter.cu, CTF_TU_FMT=1
inline cudaError_t launch_filter(const LaunchArgs &a, cudaStream_t stream) {
    if (a.filter != 0) return a.fmt == 1 ? launch_bicubic_bc1(a, stream) : launch_bicubic_mlp(a, stream);
    return a.fmt == 1 ? launch_filter_bc1(a, stream) : launch_filter_mlp(a, stream);
}

// Latent-MLP weights for the kernel parameter block, repacked from the ABI layout
// (W1[32][12] b1 W2[32][32] b2 W3[4][32] b3) into the kernels' access order (W1, b1,
// W2 transposed, b2, W3 transposed, b3).  Source: the caller's host copy (required by the
// ABI, validated non-NULL): no device round trip, no synchronisation (include/ctf.h).
inline cudaError_t mlp_weights_by_value(const LaunchArgs &a, cudaStream_t, float (&o)[kMlpParams]) {
    if (!a.mlp_host) return cudaErrorInvalidValue;
    const float *src = a.mlp_host;
    const float *W1 = src, *b1 = W1 + 384, *W2 = b1 + 32, *b2 = W2 + 1024, *W3 = b2 + 32, *b3 = W3 + 128;
    memcpy(o, W1, sizeof(float) * 384);
    memcpy(o + 384, b1, sizeof(float) * 32);
    for (int k = 0; k < 32; ++k)
        for (int j = 0; j < 32; ++j) o[416 + k * 32 + j] = W2[j * 32 + k];
    memcpy(o + 1440, b2, sizeof(float) * 32);
    for (int j = 0; j < 32; ++j)
        for (int c = 0; c < 4; ++c) o[1472 + j * 4 + c] = W3[c * 32 + j];
    memcpy(o + 1600, b3, sizeof(float) * 4);
    return cudaSuccess;
}

struct StatsDev {  // device-side accumulation, converted to ctf_frame_stats on the host
    unsigned long long waves_live, waves_partial, waves_exact, waves_fallback, waves_magnified;
    unsigned long long pixels_active, pixels_mag, evals, evals_mag;
    unsigned int max_evals_per_lane, max_unique;
    unsigned long long hist[129];
    unsigned int max_abs_err_bits;
    unsigned int pad;
    double sum_sq_err;
};

constexpr int kErrBlocks = 592;  // fixed grid => fixed (deterministic) fp64 reduction order

cudaError_t launch_stats(const uint32_t *rec, long long nrec, const float *out, const float *ref,
                         long long npix, StatsDev *dev, double *partials, cudaStream_t stream);

}  // namespace ctf
