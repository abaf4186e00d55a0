// ctf_abi.cu — the C-ABI shim (include/ctf.h): validation, launch, host pipeline.
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

#include "../../include/ctf.h"
#include "ctf_internal.h"

namespace {

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int validate(const ctf_texture *tex, const float *uv, const uint16_t *grad, int32_t Wf, int32_t Hf, int32_t frames,
             const ctf_params *p, const float *out, const uint32_t *rec) {
    if (!tex || !uv || !p || !out || !rec) return CTF_EINVAL;
    if (Wf <= 0 || Hf <= 0 || frames <= 0) return CTF_EINVAL;
    if (tex->format != CTF_FMT_BC1 && tex->format != CTF_FMT_LATENT_MLP) return CTF_EINVAL;
    if (tex->width <= 0 || tex->height <= 0 || (tex->width & 3) || (tex->height & 3)) return CTF_EINVAL;
    if (tex->addr != CTF_ADDR_CLAMP) return CTF_EINVAL;
    if (!tex->data_dev) return CTF_EINVAL;
    if (tex->format == CTF_FMT_LATENT_MLP && (!tex->mlp_dev || !tex->mlp_host)) return CTF_EINVAL;
    if (p->row0 < 0 || (p->row0 & 3) || p->reserved_ != 0) return CTF_EINVAL;
    if ((int64_t)p->row0 + Hf > (1LL << 30)) return CTF_EUNSUPPORTED;
    if (p->mode < CTF_MODE_BILINEAR_4TAP || p->mode > CTF_MODE_MASK11) return CTF_EINVAL;
    if (p->fallback < CTF_FB_STF || p->fallback > CTF_FB_CPLUS) return CTF_EINVAL;
    if (p->filter < CTF_FILTER_BILINEAR || p->filter > CTF_FILTER_CATMULL_ROM) return CTF_EINVAL;
    if (p->max_evals < 0 || p->max_evals > 2) return CTF_EINVAL;
    if (p->filter == CTF_FILTER_BILINEAR && p->max_evals > 1) return CTF_EUNSUPPORTED;
    if (p->filter != CTF_FILTER_BILINEAR) {
        // R-28: no WC estimator for signed weights; per-pixel debug outputs are bilinear-only
        if (p->mode == CTF_MODE_WAVECOMM || p->fallback == CTF_FB_WAVECOMM) return CTF_EUNSUPPORTED;
        if (p->flags & CTF_FLAG_DEBUG) return CTF_EUNSUPPORTED;
        if (!ctf::bicubic_built()) return CTF_EUNSUPPORTED;
    }
    // texel ids y*W+x must fit 24 bits (sort keys) and coordinates 16 bits
    if ((int64_t)tex->width * tex->height > (1LL << 24) || tex->width > 65535 || tex->height > 65535)
        return CTF_EUNSUPPORTED;
    // wave indices are 32-bit in the kernel
    if ((int64_t)((Wf + 7) / 8) * ((Hf + 3) / 4) * frames >= (1LL << 31)) return CTF_EUNSUPPORTED;
    // pixel indices are 32-bit in the kernel
    if ((int64_t)Wf * Hf * frames + 4LL * Wf + 8 >= (1LL << 32)) return CTF_EUNSUPPORTED;
    if (!aligned(uv, 8) || (grad && !aligned(grad, 8)) || !aligned(out, 16) || !aligned(rec, 4)) return CTF_EALIGN;
    if (!aligned(tex->data_dev, tex->format == CTF_FMT_BC1 ? 8 : 16)) return CTF_EALIGN;
    if (tex->mlp_dev && !aligned(tex->mlp_dev, 4)) return CTF_EALIGN;
    return CTF_OK;
}

ctf::LaunchArgs make_args(const ctf_texture *tex, const float *uv, const uint16_t *grad, int32_t Wf, int32_t Hf,
                          int32_t frames, const ctf_params *p, float *out, uint32_t *rec, const ctf_debug *dbg) {
    ctf::LaunchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.fmt = tex->format;
    a.W = tex->width;
    a.H = tex->height;
    a.tex_data = tex->data_dev;
    a.mlp = tex->mlp_dev;
    a.mlp_host = tex->mlp_host;
    a.uv = uv;
    a.grad = grad;
    a.Wf = Wf;
    a.Hf = Hf;
    a.frames = frames;
    a.out = out;
    a.rec = rec;
    a.mode = p->mode;
    a.fallback = p->fallback;
    a.flags = p->flags;
    a.frame_index = p->frame_index;
    a.row0 = p->row0;
    a.seed = p->seed;
    a.filter = p->filter;
    a.max_evals = p->max_evals < 1 ? 1 : p->max_evals;
    if (p->workspace_dev && p->workspace_bytes >= ctf_filter_workspace_bytes(Wf, Hf, frames) &&
        ((uintptr_t)p->workspace_dev & 15u) == 0)
        a.lists = static_cast<uint32_t *>(p->workspace_dev);
    if (dbg && (p->flags & CTF_FLAG_DEBUG)) {
        a.dbg_pid = dbg->produced_id_dev;
        a.dbg_sel = dbg->selection_dev;
        a.dbg_unread = dbg->unread_dev;
    } else {
        a.flags &= ~(uint32_t)CTF_FLAG_DEBUG;
    }
    return a;
}

}  // namespace

extern "C" {

int ctf_abi_version(void) { return CTF_ABI_VERSION; }

size_t ctf_filter_workspace_bytes(int32_t Wf, int32_t Hf, int32_t frames) {
    if (Wf <= 0 || Hf <= 0 || frames <= 0) return 0;
    const size_t waves = (size_t)((Wf + 7) / 8) * (size_t)((Hf + 3) / 4) * (size_t)frames;
    return 256 + 8 * waves;
}

int ctf_launches_per_call(int32_t format, int32_t mode, int32_t filter, int32_t Wf, int32_t Hf, int32_t frames,
                          int flags) {
    if ((format != CTF_FMT_BC1 && format != CTF_FMT_LATENT_MLP) || mode < 0 || mode > CTF_MODE_MASK11 || filter < 0 ||
        filter > 2 || Wf <= 0 || Hf <= 0 || frames < 0)
        return -1;
    const bool batched = (flags & CTF_LAUNCH_BATCHED) != 0;
    const long long waves = (long long)((Wf + 7) / 8) * ((Hf + 3) / 4) * (batched ? frames : 1);
    const int per_pass = ctf::launches_per_pass(format, mode, filter, waves,
                                                (flags & CTF_LAUNCH_SEPARATE_PASSES) ? CTF_FLAG_SEPARATE_PASSES : 0u);
    return per_pass * (batched ? (frames > 0 ? 1 : 0) : frames);
}

int ctf_filter_batch(const ctf_texture *tex, const float *uv_dev, const uint16_t *grad_dev, int32_t Wf, int32_t Hf,
                     int32_t frames, const ctf_params *p, float *out_dev, uint32_t *rec_dev, const ctf_debug *dbg,
                     void *stream) {
    const int v = validate(tex, uv_dev, grad_dev, Wf, Hf, frames, p, out_dev, rec_dev);
    if (v != CTF_OK) return v;
    const ctf::LaunchArgs a = make_args(tex, uv_dev, grad_dev, Wf, Hf, frames, p, out_dev, rec_dev, dbg);
    return ctf::launch_filter(a, static_cast<cudaStream_t>(stream)) == cudaSuccess ? CTF_OK : CTF_ECUDA;
}

int ctf_filter_frame(const ctf_texture *tex, const float *uv_dev, const uint16_t *grad_dev, int32_t Wf, int32_t Hf,
                     const ctf_params *p, float *out_dev, uint32_t *rec_dev, const ctf_debug *dbg, void *stream) {
    return ctf_filter_batch(tex, uv_dev, grad_dev, Wf, Hf, 1, p, out_dev, rec_dev, dbg, stream);
}

int ctf_stats(const uint32_t *rec_dev, int32_t Wf, int32_t Hf, int32_t frames, const float *out_dev,
              const float *ref_dev, ctf_frame_stats *host_out, void *stream) {
    if (!rec_dev || !host_out || Wf <= 0 || Hf <= 0 || frames <= 0) return CTF_EINVAL;
    if ((out_dev == nullptr) != (ref_dev == nullptr)) return CTF_EINVAL;
    if ((out_dev && !aligned(out_dev, 16)) || (ref_dev && !aligned(ref_dev, 16))) return CTF_EALIGN;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const long long nrec = (long long)((Wf + 7) / 8) * ((Hf + 3) / 4) * frames;
    const long long npix = (long long)Wf * Hf * frames;
    void *scratch = nullptr;
    const size_t bytes = sizeof(ctf::StatsDev) + sizeof(double) * ctf::kErrBlocks;
    if (cudaMallocAsync(&scratch, bytes, s) != cudaSuccess) return CTF_ECUDA;
    ctf::StatsDev *dev = static_cast<ctf::StatsDev *>(scratch);
    double *partials = reinterpret_cast<double *>(static_cast<char *>(scratch) + sizeof(ctf::StatsDev));
    ctf::StatsDev h;
    cudaError_t e = ctf::launch_stats(rec_dev, nrec, out_dev, ref_dev, npix, dev, partials, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return CTF_ECUDA;
    std::memset(host_out, 0, sizeof(*host_out));
    host_out->waves_live = h.waves_live;
    host_out->waves_partial = h.waves_partial;
    host_out->waves_exact = h.waves_exact;
    host_out->waves_fallback = h.waves_fallback;
    host_out->waves_magnified = h.waves_magnified;
    host_out->pixels_active = h.pixels_active;
    host_out->pixels_in_magnified_waves = h.pixels_mag;
    host_out->texel_evals = h.evals;
    host_out->texel_evals_in_magnified_waves = h.evals_mag;
    host_out->max_evals_per_lane = h.max_evals_per_lane;
    host_out->max_unique_per_wave = h.max_unique;
    for (int i = 0; i < 129; ++i) host_out->unique_hist[i] = h.hist[i];
    if (out_dev) {
        host_out->sum_sq_err = h.sum_sq_err;
        std::memcpy(&host_out->max_abs_err, &h.max_abs_err_bits, sizeof(float));
        host_out->err_pixels = (uint64_t)npix;
    }
    return CTF_OK;
}

size_t ctf_host_workspace_bytes(int32_t Wf, int32_t Hf, int32_t chunk_frames, int with_grad) {
    if (Wf <= 0 || Hf <= 0 || chunk_frames <= 0) return 0;
    const size_t px = (size_t)Wf * Hf * chunk_frames;
    const size_t nrec = (size_t)((Wf + 7) / 8) * ((Hf + 3) / 4) * chunk_frames;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t set = up(px * 8) + (with_grad ? up(px * 8) : 0) + up(px * 16) + up(nrec * 4);
    return 2 * set;  // double buffered
}

int ctf_filter_frames_host(const ctf_texture *tex, const float *uv_host, const uint16_t *grad_host, int32_t Wf,
                           int32_t Hf, int32_t frames, int32_t chunk_frames, const ctf_params *p, float *out_host,
                           uint32_t *rec_host, void *workspace_dev, size_t workspace_bytes, void *stream) {
    if (!tex || !uv_host || !p || !out_host || !workspace_dev || Wf <= 0 || Hf <= 0 || frames <= 0 ||
        chunk_frames <= 0)
        return CTF_EINVAL;
    if (chunk_frames > frames) chunk_frames = frames;
    const int with_grad = grad_host != nullptr;
    if (workspace_bytes < ctf_host_workspace_bytes(Wf, Hf, chunk_frames, with_grad)) return CTF_EINVAL;
    const size_t fpx = (size_t)Wf * Hf;
    const size_t frec = (size_t)((Wf + 7) / 8) * ((Hf + 3) / 4);
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t cpx = fpx * chunk_frames, crec = frec * chunk_frames;
    char *base = static_cast<char *>(workspace_dev);
    struct Set { float *uv; uint16_t *grad; float *out; uint32_t *rec; } sets[2];
    for (int b = 0; b < 2; ++b) {
        sets[b].uv = reinterpret_cast<float *>(base);
        base += up(cpx * 8);
        sets[b].grad = with_grad ? reinterpret_cast<uint16_t *>(base) : nullptr;
        base += with_grad ? up(cpx * 8) : 0;
        sets[b].out = reinterpret_cast<float *>(base);
        base += up(cpx * 16);
        sets[b].rec = reinterpret_cast<uint32_t *>(base);
        base += up(crec * 4);
    }
    cudaStream_t comp = static_cast<cudaStream_t>(stream);
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    int rc = CTF_OK;
    bool ok = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) == cudaSuccess;
    for (int b = 0; ok && b < 2; ++b)
        ok = cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev_k[b], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) rc = CTF_ECUDA;
    const int nchunks = (frames + chunk_frames - 1) / chunk_frames;
    for (int c = 0; rc == CTF_OK && c < nchunks; ++c) {
        const int b = c & 1;
        const int f0 = c * chunk_frames;
        const int nf = (f0 + chunk_frames <= frames) ? chunk_frames : frames - f0;
        Set &S = sets[b];
        bool good = true;
        if (c >= 2) good = cudaStreamWaitEvent(h2d, ev_k[b], 0) == cudaSuccess;   // inputs of chunk c-2 consumed
        good = good && cudaMemcpyAsync(S.uv, uv_host + (size_t)f0 * fpx * 2, (size_t)nf * fpx * 8,
                                       cudaMemcpyHostToDevice, h2d) == cudaSuccess;
        if (with_grad)
            good = good && cudaMemcpyAsync(S.grad, grad_host + (size_t)f0 * fpx * 4, (size_t)nf * fpx * 8,
                                           cudaMemcpyHostToDevice, h2d) == cudaSuccess;
        good = good && cudaEventRecord(ev_in[b], h2d) == cudaSuccess;
        good = good && cudaStreamWaitEvent(comp, ev_in[b], 0) == cudaSuccess;
        if (c >= 2) good = good && cudaStreamWaitEvent(comp, ev_out[b], 0) == cudaSuccess;  // outputs of c-2 drained
        if (!good) { rc = CTF_ECUDA; break; }
        ctf_params pc = *p;
        pc.frame_index = p->frame_index + (uint32_t)f0;
        pc.workspace_dev = nullptr;   // the chunks run on two streams: no shared work lists
        pc.workspace_bytes = 0;
        rc = ctf_filter_batch(tex, S.uv, S.grad, Wf, Hf, nf, &pc, S.out, S.rec, nullptr, comp);
        if (rc != CTF_OK) break;
        good = cudaEventRecord(ev_k[b], comp) == cudaSuccess && cudaStreamWaitEvent(d2h, ev_k[b], 0) == cudaSuccess;
        good = good && cudaMemcpyAsync(out_host + (size_t)f0 * fpx * 4, S.out, (size_t)nf * fpx * 16,
                                       cudaMemcpyDeviceToHost, d2h) == cudaSuccess;
        if (rec_host)
            good = good && cudaMemcpyAsync(rec_host + (size_t)f0 * frec, S.rec, (size_t)nf * frec * 4,
                                           cudaMemcpyDeviceToHost, d2h) == cudaSuccess;
        good = good && cudaEventRecord(ev_out[b], d2h) == cudaSuccess;
        if (!good) rc = CTF_ECUDA;
    }
    // every copy that reads or writes the caller's host buffers has finished before the call
    // returns — also on an error path that left the loop with H2D copies still queued
    if (h2d && cudaStreamSynchronize(h2d) != cudaSuccess) rc = CTF_ECUDA;
    if (d2h && cudaStreamSynchronize(d2h) != cudaSuccess) rc = CTF_ECUDA;
    if (cudaStreamSynchronize(comp) != cudaSuccess) rc = CTF_ECUDA;
    for (int b = 0; b < 2; ++b) {
        if (ev_in[b]) cudaEventDestroy(ev_in[b]);
        if (ev_k[b]) cudaEventDestroy(ev_k[b]);
        if (ev_out[b]) cudaEventDestroy(ev_out[b]);
    }
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    return rc;
}

}  // extern "C"
