"""Seeded texture payloads in the two synthetic formats of the hot path.

* BC1-style blocks (the paper itself uses RGBA / NTC / DCT,
  P:691-692, P:729-743, P:859-860 — the BC1-style format is ours).
  Layout: uint8[(H/4)*(W/4)*8], block-row-major; per block, little-endian
  u16 c0 @0, u16 c1 @2 (RGB565), u32 index word @4 (2 bits per texel,
  texel (x&3, y&3) at bit 2*(4*(y&3)+(x&3))).
* Latent grid + MLP weights for the NTC-style decoder:
  fp16 [H/4][W/4][8] latents and fp32 packed W1,b1,W2,b2,W3,b3 (row-major,
  W_l is [out][in]).

The encoder below picks endpoints and indices with a projection heuristic; it
contains no decode arithmetic (the decode lives separately in the oracle and
in the CUDA kernel).  All randomness is numpy's PCG64 seeded by the caller.
"""
from __future__ import annotations

import numpy as np

LATENT_CHANNELS = 8
MLP_SIZES = (12, 32, 32, 4)


def _interp_matrix(n_out: int, n_in: int) -> np.ndarray:
    """Dense linear-interpolation matrix mapping n_in grid samples to n_out."""
    pos = (np.arange(n_out) + 0.5) * (n_in - 1) / n_out
    i0 = np.clip(np.floor(pos).astype(np.int64), 0, n_in - 2)
    f = (pos - i0).astype(np.float32)
    m = np.zeros((n_out, n_in), np.float32)
    m[np.arange(n_out), i0] = 1.0 - f
    m[np.arange(n_out), i0 + 1] = f
    return m


def smooth_noise(h: int, w: int, channels: int, seed: int, octaves=(8, 32, 128)) -> np.ndarray:
    """Sum of bilinearly upsampled random grids, normalised to [0, 1]."""
    rng = np.random.default_rng(seed)
    img = np.zeros((channels, h, w), np.float32)
    amp = 1.0
    for g in octaves:
        g = max(2, min(g, h, w))
        grid = rng.random((channels, g + 1, g + 1), dtype=np.float32)
        my = _interp_matrix(h, g + 1)
        mx = _interp_matrix(w, g + 1)
        for c in range(channels):
            img[c] += amp * (my @ grid[c] @ mx.T)
        amp *= 0.5
    lo = img.min(axis=(1, 2), keepdims=True)
    hi = img.max(axis=(1, 2), keepdims=True)
    img = (img - lo) / np.maximum(hi - lo, 1e-6)
    return np.moveaxis(img, 0, -1)  # [h][w][c]


def _edges(img: np.ndarray, seed: int, count: int = 24) -> np.ndarray:
    """Overlay hard-edged rectangles so blocks see sharp colour steps."""
    rng = np.random.default_rng(seed + 7919)
    h, w, _ = img.shape
    for _ in range(count):
        x0, x1 = np.sort(rng.integers(0, w, 2))
        y0, y1 = np.sort(rng.integers(0, h, 2))
        img[y0:y1 + 1, x0:x1 + 1] = rng.random(3, dtype=np.float32)
    return img


def _to565(rgb8: np.ndarray) -> np.ndarray:
    r = (rgb8[..., 0].astype(np.uint32) * 31 + 127) // 255
    g = (rgb8[..., 1].astype(np.uint32) * 63 + 127) // 255
    b = (rgb8[..., 2].astype(np.uint32) * 31 + 127) // 255
    return (r << 11) | (g << 5) | b


def encode_bc1(rgb: np.ndarray, seed: int = 0, three_colour_frac: float = 0.03) -> np.ndarray:
    """Encode an RGB image in [0,1] ([H][W][3], H, W multiples of 4) to blocks.

    Endpoints: per-channel bounding box of the block (c0 = max, c1 = min).
    Indices: projection of each texel onto the endpoint segment (parameter
    0 at c1, 1 at c0), quantised to the 4-colour ordering {c0, c1, 2/3, 1/3}.
    A `three_colour_frac` share of blocks is written with c0 <= c1 so the
    decoder's 3-colour + transparent mode is exercised too.
    """
    h, w, _ = rgb.shape
    assert h % 4 == 0 and w % 4 == 0
    rgb8 = np.clip(np.rint(rgb * 255.0), 0, 255).astype(np.uint8)
    blk = rgb8.reshape(h // 4, 4, w // 4, 4, 3).transpose(0, 2, 1, 3, 4).reshape(-1, 16, 3)
    hi = blk.max(axis=1)
    lo = blk.min(axis=1)
    c0 = _to565(hi)
    c1 = _to565(lo)
    d = hi.astype(np.float32) - lo.astype(np.float32)
    dd = np.maximum((d * d).sum(-1, keepdims=True), 1e-6)
    t = ((blk.astype(np.float32) - lo[:, None, :].astype(np.float32)) * d[:, None, :]).sum(-1) / dd
    # t in [0,1]: 1 -> c0 (code 0), 0 -> c1 (code 1), 2/3 -> code 2, 1/3 -> code 3
    code = np.where(t > 5 / 6, 0, np.where(t < 1 / 6, 1, np.where(t >= 0.5, 2, 3))).astype(np.uint32)
    # enforce c0 > c1 for 4-colour mode; equal endpoints stay (3-colour mode, code 0 everywhere)
    swap = c0 < c1
    c0, c1 = np.where(swap, c1, c0), np.where(swap, c0, c1)
    code = np.where(swap[:, None], code ^ 1, code)  # 0<->1, 2<->3 keeps the geometry
    code = np.where((c0 == c1)[:, None], 0, code).astype(np.uint32)
    rng = np.random.default_rng(seed + 104729)
    three = rng.random(c0.shape[0]) < three_colour_frac
    c0, c1 = np.where(three, c1, c0), np.where(three, c0, c1)
    shifts = (2 * np.arange(16, dtype=np.uint32))[None, :]
    idx = np.bitwise_or.reduce(code << shifts, axis=1).astype(np.uint32)
    out = np.empty((c0.shape[0], 2), np.uint32)
    out[:, 0] = (c0 & 0xFFFF) | ((c1 & 0xFFFF) << 16)
    out[:, 1] = idx
    return out.view(np.uint8).reshape(-1).copy()


def bc1_texture(width: int, height: int, seed: int, kind: str = "image") -> np.ndarray:
    """BC1-style texture payload, uint8[(height/4)*(width/4)*8].

    kind="image": seeded smooth noise + hard edges, encoded by `encode_bc1`.
    kind="random": raw random block bytes (stress: both modes, any index).
    kind="constant": every texel decodes to one colour (c0 == c1, codes 0).
    """
    if width % 4 or height % 4:
        raise ValueError("BC1 texture dims must be multiples of 4")
    nb = (width // 4) * (height // 4)
    if kind == "random":
        return np.random.default_rng(seed).integers(0, 256, nb * 8, dtype=np.uint8)
    if kind == "constant":
        rng = np.random.default_rng(seed)
        c = np.uint32(rng.integers(0, 1 << 16))
        out = np.zeros((nb, 2), np.uint32)
        out[:, 0] = c | (c << 16)
        return out.view(np.uint8).reshape(-1).copy()
    if kind != "image":
        raise ValueError(kind)
    img = _edges(smooth_noise(height, width, 3, seed), seed)
    return encode_bc1(img, seed)


def latent_texture(width: int, height: int, seed: int) -> np.ndarray:
    """fp16 latent grid [height/4][width/4][8], smooth noise in [-1, 1]."""
    lh, lw = height // 4, width // 4
    z = smooth_noise(lh, lw, LATENT_CHANNELS, seed, octaves=(4, 16, 64)) * 2.0 - 1.0
    return z.astype(np.float16)


def mlp_weights(seed: int) -> np.ndarray:
    """Packed fp32 MLP 12->32->32->4: W1[32][12], b1[32], W2[32][32], b2[32], W3[4][32], b3[4].

    He-uniform hidden layers; the output layer is scaled down and biased to
    0.5 so most outputs land inside the [0,1] clamp.
    """
    rng = np.random.default_rng(seed)
    parts = []
    sizes = MLP_SIZES
    for li in range(3):
        fin, fout = sizes[li], sizes[li + 1]
        bound = np.sqrt(6.0 / fin)
        if li == 2:
            bound *= 0.25
        wmat = rng.uniform(-bound, bound, (fout, fin)).astype(np.float32)
        bias = rng.uniform(-0.1, 0.1, fout).astype(np.float32)
        if li == 2:
            bias += 0.5
        parts += [wmat.reshape(-1), bias]
    return np.concatenate(parts).astype(np.float32)


MLP_PARAM_COUNT = 32 * 12 + 32 + 32 * 32 + 32 + 4 * 32 + 4  # 1604
