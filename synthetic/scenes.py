"""Seeded per-pixel UV + Jacobian buffers shaped like the paper's scenes.

Buffers (the boundary's input layout, include/ctf.h):
  uv   float32 [Hf][Wf][2]   normalised texture coordinates; u = NaN marks an
                             uncovered pixel (inactive lane).
  grad float16 [Hf][Wf][4]   (du/dx, dv/dx, du/dy, dv/dy) in TEXEL units per
                             pixel; zero on uncovered pixels.

Scenes:
  G1 `rotated_quad`      — the paper's textured quad, rotated by
                           theta and magnified uniformly by m (Fig. 4's axes,
                           P:576-594); optional circle / half-plane coverage for
                           partial waves (suppl. §2 edge remapping).
  G2 `perspective_plane` — a ground plane seen by a pinhole camera with a 45°
                           vertical FOV, the shape of the teaser scene
                           (magnification ~0–9, mean ~4.3).
  `camera_path_frame`    — a 64-frame far→near→far flight over G2.

Everything is computed in float64 and rounded once to the buffer dtype, so a
given (scene, seed) always yields identical bytes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class PlaneParams:
    pitch_deg: float
    height: float
    scale: float
    yaw_deg: float = 0.0
    fov_deg: float = 45.0


# G2a: magnification ~0.9-9.1, mean ~4.3 at 1080p/2048^2 (and 4K/4096^2) — configs 2, 3, 5.
PLANE_C2 = PlaneParams(pitch_deg=40.0, height=1.0, scale=16.0)
# G2b: grazing view with horizon: strong minification + uncovered sky — config 4.
PLANE_C4 = PlaneParams(pitch_deg=20.0, height=1.0, scale=26.946)


def _pixel_grid(wf: int, hf: int):
    py, px = np.meshgrid(np.arange(hf, dtype=np.float64), np.arange(wf, dtype=np.float64), indexing="ij")
    return px, py


def _pack(u, v, jx_u, jx_v, jy_u, jy_v, covered):
    hf, wf = u.shape
    uv = np.empty((hf, wf, 2), np.float32)
    uv[..., 0] = np.where(covered, u, np.nan)
    uv[..., 1] = np.where(covered, v, np.nan)
    grad = np.zeros((hf, wf, 4), np.float16)
    grad[..., 0] = np.where(covered, jx_u, 0.0)
    grad[..., 1] = np.where(covered, jx_v, 0.0)
    grad[..., 2] = np.where(covered, jy_u, 0.0)
    grad[..., 3] = np.where(covered, jy_v, 0.0)
    return uv, grad


def rotated_quad(wf: int, hf: int, tex_w: int, tex_h: int, mag: float, theta_deg: float,
                 center=(0.5, 0.5), coverage: str | None = None, radius: float | None = None,
                 angle_deg: float = 30.0, jitter_seed: int | None = None):
    """G1: texel offset d = R(-theta) (p + 1/2 - frame/2) / mag; uv = center + d / (W, H).

    coverage: None (all covered), "circle" (pixels farther than `radius` px from
    the frame centre are uncovered), "halfplane" (pixels on one side of a line
    through the centre at `angle_deg` are uncovered).
    jitter_seed: if given, adds a seeded sub-texel offset to `center`.
    """
    th = np.deg2rad(theta_deg)
    c, s = np.cos(th), np.sin(th)
    cx, cy = center
    if jitter_seed is not None:
        r = np.random.default_rng(jitter_seed).random(2)
        cx += (r[0] - 0.5) / tex_w
        cy += (r[1] - 0.5) / tex_h
    px, py = _pixel_grid(wf, hf)
    dx = px + 0.5 - wf / 2.0
    dy = py + 0.5 - hf / 2.0
    tx = (c * dx + s * dy) / mag
    ty = (-s * dx + c * dy) / mag
    u = cx + tx / tex_w
    v = cy + ty / tex_h
    covered = np.ones_like(u, dtype=bool)
    if coverage == "circle":
        rad = radius if radius is not None else 0.45 * min(wf, hf)
        covered = dx * dx + dy * dy <= rad * rad
    elif coverage == "halfplane":
        a = np.deg2rad(angle_deg)
        covered = (np.cos(a) * dx + np.sin(a) * dy) <= 0.0
    elif coverage is not None:
        raise ValueError(coverage)
    ones = np.ones_like(u)
    return _pack(u, v, c / mag * ones, -s / mag * ones, s / mag * ones, c / mag * ones, covered)


def affine_quad(wf: int, hf: int, tex_w: int, tex_h: int, jac, center=(0.5, 0.5)):
    """A general affine mapping (anisotropic / sheared quad): texel offset d = J (p + 1/2 - frame/2),
    uv = center + d / (W, H).  `jac` = [[du/dx, du/dy], [dv/dx, dv/dy]] in texel units per pixel,
    i.e. column 0 is the texel step of one pixel along screen x, column 1 along screen y.
    grad = (du/dx, dv/dx, du/dy, dv/dy), constant."""
    J = np.asarray(jac, np.float64)
    px, py = _pixel_grid(wf, hf)
    dx = px + 0.5 - wf / 2.0
    dy = py + 0.5 - hf / 2.0
    u = center[0] + (J[0, 0] * dx + J[0, 1] * dy) / tex_w
    v = center[1] + (J[1, 0] * dx + J[1, 1] * dy) / tex_h
    ones = np.ones_like(u)
    return _pack(u, v, J[0, 0] * ones, J[1, 0] * ones, J[0, 1] * ones, J[1, 1] * ones,
                 np.ones_like(u, dtype=bool))


def _plane_uv(px, py, wf, hf, p: PlaneParams, cam_height: float):
    """Continuous pixel position -> (u, v, hit) for the ground plane z = 0."""
    t_half = np.tan(np.deg2rad(p.fov_deg) / 2.0)
    aspect = wf / hf
    xc = (2.0 * px / wf - 1.0) * t_half * aspect
    yc = (1.0 - 2.0 * py / hf) * t_half
    ph = np.deg2rad(p.pitch_deg)
    # camera looks along +Y, pitched down by `pitch`; right = +X
    fwd = np.array([0.0, np.cos(ph), -np.sin(ph)])
    up = np.array([0.0, np.sin(ph), np.cos(ph)])
    dir_y = fwd[1] + yc * up[1]
    dir_z = fwd[2] + yc * up[2]
    dir_x = xc
    hit = dir_z < -1e-12
    tt = np.where(hit, cam_height / np.where(hit, -dir_z, 1.0), 0.0)
    gx = tt * dir_x
    gy = tt * dir_y
    # pivot: the ground point under the screen centre maps to uv (0.5, 0.5)
    gyc = cam_height / np.tan(ph)
    yaw = np.deg2rad(p.yaw_deg)
    cy_, sy_ = np.cos(yaw), np.sin(yaw)
    rx = cy_ * gx - sy_ * (gy - gyc)
    ry = sy_ * gx + cy_ * (gy - gyc)
    u = 0.5 + rx / p.scale
    v = 0.5 - ry / p.scale
    return u, v, hit


def perspective_plane(wf: int, hf: int, tex_w: int, tex_h: int, params: PlaneParams = PLANE_C2,
                      cam_height: float | None = None):
    """G2: textured ground plane under a pinhole camera (45° vertical FOV).

    Pixels whose ray misses the plane or whose uv leaves [0,1]^2 are uncovered.
    grad = central differences of texel coordinates at +-0.5 px (float64).
    """
    h = params.height if cam_height is None else cam_height
    px, py = _pixel_grid(wf, hf)
    cxp, cyp = px + 0.5, py + 0.5
    u, v, hit = _plane_uv(cxp, cyp, wf, hf, params, h)
    ux1, vx1, hx1 = _plane_uv(cxp + 0.5, cyp, wf, hf, params, h)
    ux0, vx0, hx0 = _plane_uv(cxp - 0.5, cyp, wf, hf, params, h)
    uy1, vy1, hy1 = _plane_uv(cxp, cyp + 0.5, wf, hf, params, h)
    uy0, vy0, hy0 = _plane_uv(cxp, cyp - 0.5, wf, hf, params, h)
    covered = hit & hx1 & hx0 & hy1 & hy0 & (u >= 0) & (u <= 1) & (v >= 0) & (v <= 1)
    return _pack(u, v,
                 (ux1 - ux0) * tex_w, (vx1 - vx0) * tex_h,
                 (uy1 - uy0) * tex_w, (vy1 - vy0) * tex_h, covered)


def camera_path_frame(f: int, wf: int, hf: int, tex_w: int, tex_h: int, nframes: int = 64,
                      base: PlaneParams = PLANE_C2):
    """Frame f of the far->near->far flight: h_f = 1 + (1 + cos 2*pi*f/n)/2, yaw 45°*f/n."""
    hcam = 1.0 + 0.5 * (1.0 + np.cos(2.0 * np.pi * f / nframes))
    p = PlaneParams(base.pitch_deg, hcam, base.scale, 45.0 * f / nframes, base.fov_deg)
    return perspective_plane(wf, hf, tex_w, tex_h, p)


def scene_magnification(grad: np.ndarray) -> np.ndarray:
    """Descriptive statistic of an input (used only to report the scene recipe):
    m = 1 / max(|J_x|, |J_y|) in texel units, inf where the Jacobian is zero."""
    g = grad.astype(np.float64)
    jx = g[..., 0] ** 2 + g[..., 1] ** 2
    jy = g[..., 2] ** 2 + g[..., 3] ** 2
    r = np.sqrt(np.maximum(jx, jy))
    with np.errstate(divide="ignore"):
        return 1.0 / r


# ----------------------------------------------------------------------------------------------
# Device-side generation of the same scenes (torch, float64), used by bench.py to build large
# batches quickly.  Same formulas as the numpy versions above; bytes may differ in the last ulp
# of the float64 trig, so anything compared against the oracle takes host copies of these
# tensors (never regenerates them with numpy).
# ----------------------------------------------------------------------------------------------
def _plane_uv_torch(torch, px, py, wf, hf, p: PlaneParams, cam_height: float):
    import math
    t_half = math.tan(math.radians(p.fov_deg) / 2.0)
    aspect = wf / hf
    xc = (2.0 * px / wf - 1.0) * t_half * aspect
    yc = (1.0 - 2.0 * py / hf) * t_half
    ph = math.radians(p.pitch_deg)
    dir_y = math.cos(ph) + yc * math.sin(ph)
    dir_z = -math.sin(ph) + yc * math.cos(ph)
    dir_x = xc
    hit = dir_z < -1e-12
    tt = torch.where(hit, cam_height / torch.where(hit, -dir_z, torch.ones_like(dir_z)), torch.zeros_like(dir_z))
    gx = tt * dir_x
    gy = tt * dir_y
    gyc = cam_height / math.tan(ph)
    yaw = math.radians(p.yaw_deg)
    cy_, sy_ = math.cos(yaw), math.sin(yaw)
    rx = cy_ * gx - sy_ * (gy - gyc)
    ry = sy_ * gx + cy_ * (gy - gyc)
    return 0.5 + rx / p.scale, 0.5 - ry / p.scale, hit


def perspective_plane_torch(wf: int, hf: int, tex_w: int, tex_h: int, params: PlaneParams = PLANE_C2,
                            cam_height: float | None = None, device="cuda"):
    """Device twin of `perspective_plane`: returns (uv float32 [Hf][Wf][2], grad float16 [Hf][Wf][4])."""
    import torch
    h = params.height if cam_height is None else cam_height
    py, px = torch.meshgrid(torch.arange(hf, dtype=torch.float64, device=device),
                            torch.arange(wf, dtype=torch.float64, device=device), indexing="ij")
    cxp, cyp = px + 0.5, py + 0.5
    u, v, hit = _plane_uv_torch(torch, cxp, cyp, wf, hf, params, h)
    ux1, vx1, hx1 = _plane_uv_torch(torch, cxp + 0.5, cyp, wf, hf, params, h)
    ux0, vx0, hx0 = _plane_uv_torch(torch, cxp - 0.5, cyp, wf, hf, params, h)
    uy1, vy1, hy1 = _plane_uv_torch(torch, cxp, cyp + 0.5, wf, hf, params, h)
    uy0, vy0, hy0 = _plane_uv_torch(torch, cxp, cyp - 0.5, wf, hf, params, h)
    cov = hit & hx1 & hx0 & hy1 & hy0 & (u >= 0) & (u <= 1) & (v >= 0) & (v <= 1)
    nan = torch.full_like(u, float("nan"))
    uv = torch.stack([torch.where(cov, u, nan), torch.where(cov, v, nan)], -1).to(torch.float32)
    z = torch.zeros_like(u)
    grad = torch.stack([torch.where(cov, (ux1 - ux0) * tex_w, z), torch.where(cov, (vx1 - vx0) * tex_h, z),
                        torch.where(cov, (uy1 - uy0) * tex_w, z), torch.where(cov, (vy1 - vy0) * tex_h, z)],
                       -1).to(torch.float16)
    return uv.contiguous(), grad.contiguous()


def camera_path_frame_torch(f: int, wf: int, hf: int, tex_w: int, tex_h: int, nframes: int = 64,
                            base: PlaneParams = PLANE_C2, device="cuda"):
    """Device twin of `camera_path_frame`."""
    hcam = 1.0 + 0.5 * (1.0 + np.cos(2.0 * np.pi * f / nframes))
    p = PlaneParams(base.pitch_deg, hcam, base.scale, 45.0 * f / nframes, base.fov_deg)
    return perspective_plane_torch(wf, hf, tex_w, tex_h, p, device=device)
