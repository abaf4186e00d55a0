"""Test-side helpers: golden-file parsing and hand-built BC1 payloads.

Nothing here computes the method; it only lays out block bytes whose decoded
values follow by hand from the format definition (R-9).
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_rows(name: str):
    rows = []
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append(line.split())
    return rows


def blocks_from(c0: np.ndarray, c1: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Pack per-block (c0, c1, index word) arrays into the uint8 block payload."""
    b = np.empty((c0.size, 2), np.uint32)
    b[:, 0] = (c0.reshape(-1).astype(np.uint32) & 0xFFFF) | ((c1.reshape(-1).astype(np.uint32) & 0xFFFF) << 16)
    b[:, 1] = idx.reshape(-1).astype(np.uint32)
    return b.view(np.uint8).reshape(-1).copy()


def codes_word(codes_4x4) -> int:
    """Index word from codes[y][x] (2 bits per texel at 2*(4y+x))."""
    w = 0
    for y in range(4):
        for x in range(4):
            w |= (int(codes_4x4[y][x]) & 3) << (2 * (4 * y + x))
    return w


def ramp_texture(axis: str = "x", height: int = 16):
    """16-texel green ramp: G8(k) = 4k for k = texel index along `axis` (0..15).

    Block b along the axis uses c1.g6 = 4b (-> G8 = 16b) and c0.g6 = 4b+3
    (-> G8 = 16b+12, since g6 < 16 replicates as g6<<2); codes along the axis
    (1, 3, 2, 0) give 16b + {0, 4, 8, 12}: (c0+2c1)/3 = 16b+4, (2c0+c1)/3 = 16b+8
    exactly.  Red = blue = 0 (c0.r = c1.r = 0), alpha = 255 (c0 > c1).
    Returns (tex dict, W, H).
    """
    order = [1, 3, 2, 0]
    if axis == "x":
        W, H = 16, height
        nbx, nby = 4, H // 4
        c0 = np.zeros((nby, nbx), np.uint32)
        c1 = np.zeros((nby, nbx), np.uint32)
        for bx in range(nbx):
            c0[:, bx] = (4 * bx + 3) << 5
            c1[:, bx] = (4 * bx) << 5
        word = codes_word([[order[x] for x in range(4)] for _ in range(4)])
    else:
        W, H = height, 16
        nbx, nby = W // 4, 4
        c0 = np.zeros((nby, nbx), np.uint32)
        c1 = np.zeros((nby, nbx), np.uint32)
        for by in range(nby):
            c0[by, :] = (4 * by + 3) << 5
            c1[by, :] = (4 * by) << 5
        word = codes_word([[order[y]] * 4 for y in range(4)])
    idx = np.full(c0.shape, word, np.uint32)
    return {"format": 1, "width": W, "height": H, "bc1": blocks_from(c0, c1, idx)}, W, H


def bc1_tex(width: int, height: int, seed: int, kind: str = "image"):
    import synthetic
    return {"format": 1, "width": width, "height": height, "bc1": synthetic.bc1_texture(width, height, seed, kind)}


def mlp_tex(width: int, height: int, seed: int):
    import synthetic
    return {"format": 2, "width": width, "height": height,
            "latent": synthetic.latent_texture(width, height, seed), "mlp": synthetic.mlp_weights(seed + 1)}
