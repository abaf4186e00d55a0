// ctf_internal.h — launcher interface between the C-ABI shim and the kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ctf {

constexpr int kMlpParams = 32 * 12 + 32 + 32 * 32 + 32 + 4 * 32 + 4;  // 1604 (R-10)

struct LaunchArgs {
    // texture
    int fmt, W, H;
    const void *tex_data;   // BC1 blocks or fp16 latents
    const float *mlp;       // device copy of the MLP weights
    const float *mlp_host;  // optional host copy (passed by value to the kernel)
    // frames
    const float *uv;        // [frames][Hf][Wf][2]
    const uint16_t *grad;   // [frames][Hf][Wf][4] fp16 bits or nullptr
    int Wf, Hf, frames;
    float *out;             // [frames][Hf][Wf][4]
    uint32_t *rec;          // [frames][nwy][nwx]
    // parameters
    int mode, fallback;
    uint32_t flags, frame_index;
    uint64_t seed;
    // debug
    uint32_t *dbg_pid, *dbg_sel, *dbg_unread;
};

cudaError_t launch_filter_bc1(const LaunchArgs &a, cudaStream_t stream);  // ctf_filter.cu, CTF_TU_FMT=1
cudaError_t launch_filter_mlp(const LaunchArgs &a, cudaStream_t stream);  // ctf_filter.cu, CTF_TU_FMT=2
inline cudaError_t launch_filter(const LaunchArgs &a, cudaStream_t stream) {
    return a.fmt == 1 ? launch_filter_bc1(a, stream) : launch_filter_mlp(a, stream);
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
