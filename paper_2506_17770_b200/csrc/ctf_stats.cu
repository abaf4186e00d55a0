// ctf_stats.cu — frame/batch totals from per-wave records and the
// error of a filtered frame against a reference (PSNR inputs).
// Integer counters use atomics (order-independent); the fp64 sum of squared
// errors is reduced in a fixed order (fixed grid, per-block tree, single-block
// final pass), so results are bitwise reproducible.
#include <cstdint>

#include "ctf_internal.h"

namespace ctf {

constexpr int kStatThreads = 256;

__global__ void __launch_bounds__(kStatThreads) stats_records_kernel(const uint32_t *__restrict__ rec, long long nrec,
                                                                     StatsDev *__restrict__ st) {
    __shared__ unsigned long long hist[129];
    for (int i = threadIdx.x; i < 129; i += blockDim.x) hist[i] = 0ull;
    __syncthreads();
    unsigned long long live = 0, partial = 0, exact = 0, fb = 0, mag = 0, pix = 0, pixmag = 0, ev = 0, evmag = 0;
    unsigned int maxl = 0, maxn = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t r = rec[i];
        const uint32_t e = (r & 0xFFu) | (((r >> 27) & 7u) << 8), n = (r >> 8) & 0xFFu, a = (r >> 16) & 0x3Fu, path = (r >> 22) & 7u;
        const uint32_t m = (r >> 25) & 1u, p = (r >> 26) & 1u;
        if (a == 0) continue;
        ++live;
        partial += p;
        exact += (path == 0);
        fb += (path >= 1 && path <= 4);
        pix += a;
        ev += e;
        if (m) { ++mag; pixmag += a; evmag += e; }
        const unsigned int per_lane = (e + a - 1u) / a;  // ceil(evals / a): 4TAP 4 (16 bicubic), else 1-2
        maxl = max(maxl, per_lane);
        if (n <= 128) {
            maxn = max(maxn, n);
            atomicAdd(&hist[n], 1ull);
        }
    }
    // warp reduce then one atomic per warp
    for (int d = 16; d > 0; d >>= 1) {
        live += __shfl_down_sync(0xffffffffu, live, d);
        partial += __shfl_down_sync(0xffffffffu, partial, d);
        exact += __shfl_down_sync(0xffffffffu, exact, d);
        fb += __shfl_down_sync(0xffffffffu, fb, d);
        mag += __shfl_down_sync(0xffffffffu, mag, d);
        pix += __shfl_down_sync(0xffffffffu, pix, d);
        pixmag += __shfl_down_sync(0xffffffffu, pixmag, d);
        ev += __shfl_down_sync(0xffffffffu, ev, d);
        evmag += __shfl_down_sync(0xffffffffu, evmag, d);
        maxl = max(maxl, __shfl_down_sync(0xffffffffu, maxl, d));
        maxn = max(maxn, __shfl_down_sync(0xffffffffu, maxn, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&st->waves_live, live);
        atomicAdd(&st->waves_partial, partial);
        atomicAdd(&st->waves_exact, exact);
        atomicAdd(&st->waves_fallback, fb);
        atomicAdd(&st->waves_magnified, mag);
        atomicAdd(&st->pixels_active, pix);
        atomicAdd(&st->pixels_mag, pixmag);
        atomicAdd(&st->evals, ev);
        atomicAdd(&st->evals_mag, evmag);
        atomicMax(&st->max_evals_per_lane, maxl);
        atomicMax(&st->max_unique, maxn);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 129; i += blockDim.x)
        if (hist[i]) atomicAdd(&st->hist[i], hist[i]);
}

__global__ void __launch_bounds__(kStatThreads) stats_error_kernel(const float4 *__restrict__ out,
                                                                   const float4 *__restrict__ ref, long long npix,
                                                                   double *__restrict__ partials,
                                                                   StatsDev *__restrict__ st) {
    __shared__ double red[kStatThreads];
    double acc = 0.0;
    float mx = 0.0f;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (long long)gridDim.x * blockDim.x) {
        const float4 o = out[i], r = ref[i];
        const double d0 = (double)o.x - r.x, d1 = (double)o.y - r.y, d2 = (double)o.z - r.z, d3 = (double)o.w - r.w;
        acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(o.x - r.x), fabsf(o.y - r.y)), fmaxf(fabsf(o.z - r.z), fabsf(o.w - r.w))));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kStatThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
    for (int d = 16; d > 0; d >>= 1) mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, d));
    if ((threadIdx.x & 31) == 0) atomicMax(&st->max_abs_err_bits, __float_as_uint(mx));  // mx >= 0
}

__global__ void stats_error_final_kernel(const double *__restrict__ partials, int n, StatsDev *__restrict__ st) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += partials[i];
        st->sum_sq_err = s;
    }
}

cudaError_t launch_stats(const uint32_t *rec, long long nrec, const float *out, const float *ref, long long npix,
                         StatsDev *dev, double *partials, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(dev, 0, sizeof(StatsDev), stream);
    if (e != cudaSuccess) return e;
    long long blocks = (nrec + kStatThreads - 1) / kStatThreads;
    if (blocks > 1184) blocks = 1184;
    if (blocks < 1) blocks = 1;
    stats_records_kernel<<<(unsigned)blocks, kStatThreads, 0, stream>>>(rec, nrec, dev);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (out && ref) {
        stats_error_kernel<<<kErrBlocks, kStatThreads, 0, stream>>>(reinterpret_cast<const float4 *>(out),
                                                                   reinterpret_cast<const float4 *>(ref), npix,
                                                                   partials, dev);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        stats_error_final_kernel<<<1, 32, 0, stream>>>(partials, kErrBlocks, dev);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ctf
