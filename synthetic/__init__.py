"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This package is the ONLY code both sides share.  It holds no arithmetic of the
method (no footprint, dedupe, decode, RNG draw or filtering): it only writes
the bytes that go INTO `ctf_filter_frame` / the oracle — per-pixel UV and
Jacobian buffers shaped like the paper's scenes (§4 / suppl. §3.1,
P:1401-1434) and texture payloads in the synthetic formats (BC1-style blocks,
latent grid + MLP weights).  The recipe is stated in DESIGN.md §"Inputs".
"""
from .scenes import (  # noqa: F401
    rotated_quad,
    affine_quad,
    perspective_plane,
    camera_path_frame,
    camera_path_frame_torch,
    perspective_plane_torch,
    scene_magnification,
    PLANE_C2,
    PLANE_C4,
)
from .textures import bc1_texture, latent_texture, mlp_weights  # noqa: F401
