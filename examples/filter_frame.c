/*
 * filter_frame.c — the C ABI (include/ctf.h) from plain C99, no Python.
 *
 *   gcc -std=c99 -O2 -I include -I /usr/local/cuda/include examples/filter_frame.c \
 *       -L paper_2506_17770_b200 -lctf -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2506_17770_b200 -o /tmp/ctf_example && /tmp/ctf_example
 *
 * Builds a 64 x 64 BC1-style texture on the host whose 4 x 4 blocks are each one flat colour
 * (c0 = c1, every code 0: the block's texels all decode to c0), magnifies it 4x onto a
 * 96 x 40 frame (a ragged right / bottom edge) with the last column uncovered (u = NaN), and
 * filters it with the collaborative List method + C+ fallback.  Checks, from the format and
 * the method alone: the argument validation of the ABI (before any device work), every
 * covered pixel inside a block's interior equals the block colour (bilinear of equal texels),
 * uncovered pixels are (0,0,0,0), and every live wave is exact (magnification 4: n <= 32).
 * Exit status 0 = pass, 1 = fail, 77 = no CUDA device (only the validation checks ran).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "ctf.h"

#define TW 64
#define TH 64
#define WF 96
#define HF 40

static int fails = 0;
#define CHECK(cond, ...)                      \
    do {                                      \
        if (!(cond)) {                        \
            fprintf(stderr, "FAIL: " __VA_ARGS__); \
            fputc('\n', stderr);              \
            ++fails;                          \
        }                                     \
    } while (0)

/* RGB565 of block (bx, by): a flat colour per block */
static uint16_t block_colour(int bx, int by) {
    const unsigned r = (unsigned)(bx * 2) & 31u, g = (unsigned)(by * 4) & 63u, b = (unsigned)(bx + by) & 31u;
    return (uint16_t)((r << 11) | (g << 5) | b);
}

/* 565 -> 888 by bit replication, / 255 (R-9) */
static void decode565(uint16_t c, float rgba[4]) {
    const unsigned r = (c >> 11) & 31u, g = (c >> 5) & 63u, b = c & 31u;
    rgba[0] = (float)((r << 3) | (r >> 2)) / 255.0f;
    rgba[1] = (float)((g << 2) | (g >> 4)) / 255.0f;
    rgba[2] = (float)((b << 3) | (b >> 2)) / 255.0f;
    rgba[3] = 1.0f;
}

int main(void) {
    /* host texture: (TH/4) x (TW/4) blocks of 8 bytes, c0 = c1 = the block colour, codes 0 */
    static uint8_t blocks[(TH / 4) * (TW / 4) * 8];
    for (int by = 0; by < TH / 4; ++by)
        for (int bx = 0; bx < TW / 4; ++bx) {
            uint8_t *p = blocks + 8 * (by * (TW / 4) + bx);
            const uint16_t c = block_colour(bx, by);
            p[0] = (uint8_t)(c & 0xFF); p[1] = (uint8_t)(c >> 8);
            p[2] = p[0]; p[3] = p[1];
            p[4] = p[5] = p[6] = p[7] = 0;
        }
    /* uv: pixel (x, y) -> texel position (8 + x / 4, 8 + y / 4) + 1/8 (magnification 4) */
    static float uv[HF][WF][2] __attribute__((aligned(16)));
    for (int y = 0; y < HF; ++y)
        for (int x = 0; x < WF; ++x) {
            uv[y][x][0] = (x == WF - 1) ? NAN : (8.0f + (x + 0.5f) / 4.0f) / TW;
            uv[y][x][1] = (8.0f + (y + 0.5f) / 4.0f) / TH;
        }

    /* 1. validation runs on the host before anything is enqueued (no device needed) */
    ctf_params prm;
    memset(&prm, 0, sizeof(prm));
    prm.mode = CTF_MODE_COLLAB;
    prm.fallback = CTF_FB_CPLUS;
    prm.seed = 7;
    ctf_texture tex;
    memset(&tex, 0, sizeof(tex));
    tex.format = CTF_FMT_BC1;
    tex.width = TW;
    tex.height = TH;
    tex.addr = CTF_ADDR_CLAMP;
    float dummy_out[4] __attribute__((aligned(16)));
    uint32_t dummy_rec[1];
    CHECK(ctf_abi_version() == CTF_ABI_VERSION, "ABI version %d", ctf_abi_version());
    CHECK(ctf_filter_frame(NULL, &uv[0][0][0], NULL, WF, HF, &prm, dummy_out, dummy_rec, NULL, NULL) == CTF_EINVAL,
          "NULL texture must be CTF_EINVAL");
    CHECK(ctf_filter_frame(&tex, &uv[0][0][0], NULL, WF, HF, &prm, dummy_out, dummy_rec, NULL, NULL) == CTF_EINVAL,
          "NULL texture data must be CTF_EINVAL");
    tex.width = 62;
    tex.data_dev = blocks;
    CHECK(ctf_filter_frame(&tex, &uv[0][0][0], NULL, WF, HF, &prm, dummy_out, dummy_rec, NULL, NULL) == CTF_EINVAL,
          "width not a multiple of 4 must be CTF_EINVAL");
    tex.width = TW;
    prm.mode = 42;
    CHECK(ctf_filter_frame(&tex, &uv[0][0][0], NULL, WF, HF, &prm, dummy_out, dummy_rec, NULL, NULL) == CTF_EINVAL,
          "unknown mode must be CTF_EINVAL");
    prm.mode = CTF_MODE_COLLAB;
    CHECK(ctf_filter_frame(&tex, &uv[0][0][0], NULL, WF, HF, &prm, dummy_out + 1, dummy_rec, NULL, NULL) == CTF_EALIGN,
          "misaligned out must be CTF_EALIGN");
    CHECK(ctf_filter_workspace_bytes(WF, HF, 1) == 256 + 8 * (size_t)((WF + 7) / 8) * ((HF + 3) / 4),
          "workspace size");
    CHECK(ctf_launches_per_call(CTF_FMT_BC1, CTF_MODE_COLLAB, CTF_FILTER_BILINEAR, WF, HF, 1, 0) >= 1,
          "launch count");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        printf("validation checks: %s; no CUDA device, filtering skipped\n", fails ? "FAILED" : "ok");
        return fails ? 1 : 77;
    }

    /* 2. device buffers (owned by the caller), one frame filtered asynchronously on a stream */
    const int nwx = (WF + 7) / 8, nwy = (HF + 3) / 4;
    void *d_blocks = NULL, *d_uv = NULL, *d_out = NULL, *d_rec = NULL;
    cudaStream_t stream = NULL;
    int ok = cudaMalloc(&d_blocks, sizeof(blocks)) == cudaSuccess && cudaMalloc(&d_uv, sizeof(uv)) == cudaSuccess &&
             cudaMalloc(&d_out, sizeof(float) * 4 * WF * HF) == cudaSuccess &&
             cudaMalloc(&d_rec, sizeof(uint32_t) * nwx * nwy) == cudaSuccess &&
             cudaStreamCreate(&stream) == cudaSuccess &&
             cudaMemcpy(d_blocks, blocks, sizeof(blocks), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(d_uv, uv, sizeof(uv), cudaMemcpyHostToDevice) == cudaSuccess;
    CHECK(ok, "device allocation / upload");
    if (!ok) return 1;
    tex.data_dev = d_blocks;
    int rc = ctf_filter_frame(&tex, (const float *)d_uv, NULL, WF, HF, &prm, (float *)d_out, (uint32_t *)d_rec,
                              NULL, stream);
    CHECK(rc == CTF_OK, "ctf_filter_frame returned %d", rc);
    ctf_frame_stats st;
    rc = ctf_stats((const uint32_t *)d_rec, WF, HF, 1, NULL, NULL, &st, stream);   /* synchronises */
    CHECK(rc == CTF_OK, "ctf_stats returned %d", rc);

    static float out[HF][WF][4];
    static uint32_t rec[(HF + 3) / 4][(WF + 7) / 8];
    CHECK(cudaMemcpy(out, d_out, sizeof(out), cudaMemcpyDeviceToHost) == cudaSuccess, "download out");
    CHECK(cudaMemcpy(rec, d_rec, sizeof(rec), cudaMemcpyDeviceToHost) == cudaSuccess, "download records");

    /* 3. checks from the format and the method alone */
    int interior = 0;
    for (int y = 0; y < HF; ++y)
        for (int x = 0; x < WF; ++x) {
            if (x == WF - 1) {
                CHECK(out[y][x][0] == 0.0f && out[y][x][1] == 0.0f && out[y][x][2] == 0.0f && out[y][x][3] == 0.0f,
                      "uncovered pixel (%d, %d) not zero", x, y);
                continue;
            }
            /* footprint texels x0 = floor(fx - 0.5) .. x0 + 1: inside one block -> flat colour */
            const float fx = 8.0f + (x + 0.5f) / 4.0f - 0.5f, fy = 8.0f + (y + 0.5f) / 4.0f - 0.5f;
            const int x0 = (int)floorf(fx), y0 = (int)floorf(fy);
            if ((x0 >> 2) != ((x0 + 1) >> 2) || (y0 >> 2) != ((y0 + 1) >> 2)) continue;
            float ref[4];
            decode565(block_colour(x0 >> 2, y0 >> 2), ref);
            for (int c = 0; c < 4; ++c)
                CHECK(fabsf(out[y][x][c] - ref[c]) <= 1e-6f, "pixel (%d, %d) channel %d: %g vs %g", x, y, c,
                      out[y][x][c], ref[c]);
            ++interior;
        }
    for (int wy = 0; wy < nwy; ++wy)
        for (int wx = 0; wx < nwx; ++wx) {
            const uint32_t r = rec[wy][wx];
            CHECK(CTF_REC_PATH(r) == 0 && CTF_REC_N(r) <= CTF_REC_A(r), "wave (%d, %d) not exact: rec %08x", wx, wy,
                  (unsigned)r);
        }
    CHECK(st.waves_live == (uint64_t)nwx * nwy && st.waves_exact == st.waves_live && st.waves_fallback == 0,
          "stats: live %llu exact %llu", (unsigned long long)st.waves_live, (unsigned long long)st.waves_exact);
    CHECK(st.pixels_active == (uint64_t)(WF - 1) * HF, "stats: active pixels %llu", (unsigned long long)st.pixels_active);
    printf("%d interior pixels checked; %.3f texel evaluations per pixel (4-tap: 4); %s\n", interior,
           (double)st.texel_evals / (double)st.pixels_active, fails ? "FAILED" : "ok");
    cudaStreamDestroy(stream);
    cudaFree(d_blocks);
    cudaFree(d_uv);
    cudaFree(d_out);
    cudaFree(d_rec);
    return fails ? 1 : 0;
}
