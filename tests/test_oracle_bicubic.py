"""Pins of the oracle's bicubic filters (§5.4; R-24..R-28).

Everything here is checked against closed forms of the cubic B-spline / Catmull-Rom
kernels (moments, interpolation, linear reproduction), brute force on tiny frames, or
expectations of the stochastic estimators — never against the oracle itself.
"""
from __future__ import annotations

import numpy as np
import pytest

import synthetic
from oracle import oracle
from oracle.oracle import (FB_C, FB_CPLUS, FB_STF, FILTER_BSPLINE, FILTER_CATMULL_ROM, FL_FORCE_FALLBACK,
                           M_4TAP, M_BOX, M_COLLAB, M_MASK11, M_MASK16, M_STF, decode_record, filter_frame)
from tests.helpers import bc1_tex, ramp_texture

FILTERS = [FILTER_BSPLINE, FILTER_CATMULL_ROM]


# ------------------------------------------------------------ weights: closed forms --
def test_cubic_weights_closed_forms():
    """Uniform cubic B-spline: (1, 4, 1, 0)/6 at s = 0, weights >= 0, variance 1/3.
    Catmull-Rom: (0, 1, 0, 0) at s = 0 (interpolating), (-1, 9, 9, -1)/16 at s = 1/2,
    quadratic precision.  Both: partition of unity, symmetry w_i(s) = w_{3-i}(1-s) and
    linear precision sum_i w_i (i - 1) = s.  (Textbook moments of the two kernels.)"""
    b0 = oracle.cubic_weights(FILTER_BSPLINE, 0.0)
    np.testing.assert_allclose(b0, [1 / 6, 4 / 6, 1 / 6, 0.0], rtol=0, atol=6e-8)
    assert np.array_equal(oracle.cubic_weights(FILTER_CATMULL_ROM, 0.0), np.float32([0, 1, 0, 0]))
    assert np.array_equal(oracle.cubic_weights(FILTER_CATMULL_ROM, 0.5),
                          np.float32([-1 / 16, 9 / 16, 9 / 16, -1 / 16]))
    rng = np.random.default_rng(3)
    off = np.arange(4) - 1.0
    for s in np.concatenate([rng.random(400), [0.25, 0.75, 1 - 2 ** -24]]).astype(np.float32):
        for f in FILTERS:
            w = oracle.cubic_weights(f, float(s)).astype(np.float64)
            wm = oracle.cubic_weights(f, float(np.float32(1) - s)).astype(np.float64)
            assert abs(w.sum() - 1.0) < 4e-7
            np.testing.assert_allclose(w, wm[::-1], atol=3e-7)
            assert abs((w * off).sum() - float(s)) < 1e-6                       # linear precision
            second = (w * (off - float(s)) ** 2).sum()
            if f == FILTER_BSPLINE:
                assert np.all(w >= 0) and abs(second - 1.0 / 3.0) < 1e-6          # B-spline variance
            else:
                assert abs(second) < 1e-6                                         # CR: quadratic precision
                assert w[0] <= 0 and w[3] <= 0 and w[1] >= 0 and w[2] >= 0


def _fx(coord: np.ndarray, dim: int) -> np.ndarray:
    """fx = clamp(u, 0, 1) * dim - 0.5 in fp32 (dim a power of two: the product is exact,
    so this equals the single-rounding fma of R-2 / R-24)."""
    c = np.clip(coord.astype(np.float32), np.float32(0), np.float32(1))
    return (c * np.float32(dim)).astype(np.float32) - np.float32(0.5)


# --------------------------------------------- exact path: linear-ramp closed form --
@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("mode", [M_4TAP, M_COLLAB])
def test_bicubic_linear_ramp_closed_form(filt, axis, mode):
    """Both kernels reproduce linear functions (linear precision), so on the ramp
    G8(k) = 4k the filtered green is 4 f / 255 wherever all 4 taps lie inside the
    texture (1 <= f < 13): the 16-tap filter and every exact collaborative wave."""
    tex, W, H = ramp_texture(axis, height=16)
    wf, hf = 40, 20
    py, px = np.mgrid[0:hf, 0:wf].astype(np.float64)
    uv = np.empty((hf, wf, 2), np.float32)
    uv[..., 0] = (px * 0.29 + py * 0.07) / W + 0.02
    uv[..., 1] = (py * 0.27 - px * 0.05) / H + 0.3
    r = filter_frame(tex, uv, None, mode, FB_STF, filter=filt, max_evals=2, debug=False)
    d = decode_record(r["rec"])
    f = _fx(uv[..., 0] if axis == "x" else uv[..., 1], W if axis == "x" else H).astype(np.float64)
    inside = (f >= 1.0) & (f < 13.0)
    ok = np.repeat(np.repeat(d["path"] == (0 if mode == M_COLLAB else 5), 4, 0), 8, 1)[:hf, :wf] & inside
    assert ok.sum() > 100
    np.testing.assert_allclose(r["out"][..., 1][ok], 4.0 * f[ok] / 255.0, atol=2e-6)
    np.testing.assert_allclose(r["out"][..., 3][ok], 1.0, atol=1e-6)


# ----------------------------------------------- texel centres: interpolation / smoothing --
def test_texel_centres_catmull_rom_interpolates_bspline_smooths():
    """At texel centres (s = t = 0) Catmull-Rom returns the texel itself and the B-spline
    the separable [1 4 1]/6 x [1 4 1]/6 average (closed forms of the two kernels)."""
    W = H = 16
    tex = bc1_tex(W, H, 5, "random")
    val = np.array([[oracle.bc1_texel(tex["bc1"], W, x, y) for x in range(W)] for y in range(H)],
                   np.float64) / 255.0
    ys, xs = np.mgrid[2:14, 3:13]
    uv = np.stack([(xs + 0.5) / W, (ys + 0.5) / H], -1).astype(np.float32)
    cr = filter_frame(tex, uv, None, M_4TAP, filter=FILTER_CATMULL_ROM, debug=False)["out"]
    np.testing.assert_array_equal(cr, val[ys, xs])
    bs = filter_frame(tex, uv, None, M_4TAP, filter=FILTER_BSPLINE, debug=False)["out"]
    k = np.array([1.0, 4.0, 1.0]) / 6.0
    expect = sum(k[j] * k[i] * val[ys + j - 1, xs + i - 1] for j in range(3) for i in range(3))
    np.testing.assert_allclose(bs, expect, atol=2e-7)


# ---------------------------------------------- unique set and decision: brute force --
@pytest.mark.parametrize("E", [1, 2])
def test_bicubic_unique_count_and_decision_brute_force(E):
    """n = |union of the active 4x4 clamped footprints| (List semantics), recorded
    saturated at E*a + 1 (R-28); exact iff n <= E*a; evals = n when exact."""
    rng = np.random.default_rng(11 + E)
    W = H = 32
    tex = bc1_tex(W, H, 1, "random")
    paths = set()
    for trial in range(6):
        wf, hf = 19, 9
        if trial < 4:   # random per-pixel coordinates in a box of varying size
            scale = [0.12, 0.3, 1.0, 0.06][trial]
            uv = (rng.random((hf, wf, 2)) * scale + rng.random(2) * (1 - scale)).astype(np.float32)
        else:           # smooth magnified mapping (m ~ 2.5 / 4), touching the texture edge
            py, px = np.mgrid[0:hf, 0:wf].astype(np.float64)
            m = [2.5, 4.0][trial - 4]
            uv = np.stack([(px * 0.9 + py * 0.4) / (m * W) - 0.02, (py * 0.9 - px * 0.4) / (m * H) + 0.4],
                          -1).astype(np.float32)
        uv[rng.random((hf, wf)) < 0.2, 0] = np.nan
        r = filter_frame(tex, uv, None, M_COLLAB, FB_C, seed=trial, filter=FILTER_CATMULL_ROM, max_evals=E,
                         debug=False)
        d = decode_record(r["rec"])
        fx, fy = _fx(uv[..., 0], W), _fx(uv[..., 1], H)
        for wy in range(d["n"].shape[0]):
            for wx in range(d["n"].shape[1]):
                ids, a = set(), 0
                for ly in range(4):
                    for lx in range(8):
                        x, y = wx * 8 + lx, wy * 4 + ly
                        if x < wf and y < hf and not np.isnan(uv[y, x, 0]):
                            a += 1
                            x0, y0 = int(np.floor(fx[y, x])), int(np.floor(fy[y, x]))
                            for j in range(4):
                                for i in range(4):
                                    ids.add(min(max(y0 - 1 + j, 0), H - 1) * W + min(max(x0 - 1 + i, 0), W - 1))
                n = len(ids)
                assert d["a"][wy, wx] == a
                if a == 0:
                    continue
                assert d["n"][wy, wx] == min(n, E * a + 1)
                assert d["path"][wy, wx] == (0 if n <= E * a else 3)
                paths.add(int(d["path"][wy, wx]))
                if n <= E * a:
                    assert d["evals"][wy, wx] == n
    assert paths == {0, 3}


# ------------------------------------------------ stochastic estimators: expectations --
@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("which", ["positivized", "one_tap"])
def test_bicubic_stf_expectation(filt, which):
    """Positivized STF (W+ p+ - W- p-) and the fallbacks' one-tap sample
    (sign(w) sum|w| p with P = |w| / sum|w|) are unbiased: their mean over
    independent draws converges to the 16-tap filter."""
    W = H = 16
    tex = bc1_tex(W, H, 6, "random")
    uv = np.empty((32, 64, 2), np.float32)
    uv[..., 0], uv[..., 1] = 6.8 / W, 9.35 / H
    ref = filter_frame(tex, uv[:1, :1], None, M_4TAP, filter=filt)["out"][0, 0]
    acc, nfr = np.zeros(4), 24
    for f in range(nfr):
        if which == "positivized":
            o = filter_frame(tex, uv, None, M_STF, seed=77, frame_index=f, filter=filt, debug=False)["out"]
        else:
            o = filter_frame(tex, uv, None, M_COLLAB, FB_STF, FL_FORCE_FALLBACK, seed=77, frame_index=f,
                             filter=filt, debug=False)["out"]
        acc += o.mean((0, 1))
    acc /= nfr
    # 49152 draws; |estimate| <= sum|w| <= 1.6 for Catmull-Rom -> std of the mean < 8e-3
    np.testing.assert_allclose(acc, ref, atol=2.5e-2 if filt == FILTER_CATMULL_ROM else 1e-2)


def test_positivized_stf_evaluations():
    """Positivization draws one texel per lobe: 2 per pixel when the footprint
    has negative weights (Catmull-Rom off texel centres), 1 for the B-spline."""
    W = H = 64
    tex = bc1_tex(W, H, 2, "random")
    uv, _ = synthetic.rotated_quad(32, 16, W, H, 3.0, 20.0)
    a = (~np.isnan(uv[..., 0])).sum()
    cr = decode_record(filter_frame(tex, uv, None, M_STF, filter=FILTER_CATMULL_ROM, debug=False)["rec"])
    bs = decode_record(filter_frame(tex, uv, None, M_STF, filter=FILTER_BSPLINE, debug=False)["rec"])
    assert cr["evals"].sum() == 2 * a and bs["evals"].sum() == a


# ---------------------------------------------------- Eq. 1 invariants / constant texture --
@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("mode,fb,flags", [(M_4TAP, 0, 0), (M_STF, 0, 0), (M_COLLAB, FB_C, FL_FORCE_FALLBACK),
                                           (M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK), (M_COLLAB, FB_CPLUS, 0),
                                           (M_BOX, FB_C, 0), (M_MASK16, FB_CPLUS, 0)])
def test_bicubic_constant_texture(filt, mode, fb, flags):
    """Partition of unity, Eq. 1's weights and W+ - W- = sum w make every deterministic-
    weight estimator return a constant texture exactly (to fp32 weight rounding)."""
    tex = bc1_tex(64, 64, 3, "constant")
    uv, g = synthetic.rotated_quad(37, 21, 64, 64, 1.3, 33.0, coverage="circle", radius=9.0)
    r = filter_frame(tex, uv, g, mode, fb, flags, seed=9, filter=filt, debug=False)
    cov = ~np.isnan(uv[..., 0])
    c = r["out"][cov]
    np.testing.assert_allclose(c, np.broadcast_to(c[0], c.shape), atol=2e-6)
    assert np.all(r["out"][~cov] == 0.0)


def test_bicubic_eq1_special_cases_and_convexity():
    """C (Eq. 1): a lane whose known set holds every nonzero-weight texel returns the exact
    filter; otherwise its colour lies in the range Eq. 1 allows (convex in the B-spline
    case, where all weights are >= 0)."""
    W = H = 64
    tex = bc1_tex(W, H, 4, "image")
    uv, _ = synthetic.rotated_quad(48, 24, W, H, 1.4, 25.0)
    ex = filter_frame(tex, uv, None, M_4TAP, filter=FILTER_BSPLINE, debug=False)["out"]
    r = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=5, filter=FILTER_BSPLINE,
                     debug=False)["out"]
    val = np.array([[oracle.bc1_texel(tex["bc1"], W, x, y) for x in range(W)] for y in range(H)]) / 255.0
    fx, fy = _fx(uv[..., 0], W), _fx(uv[..., 1], H)
    same = 0
    for y in range(uv.shape[0]):
        for x in range(uv.shape[1]):
            x0, y0 = int(np.floor(fx[y, x])), int(np.floor(fy[y, x]))
            xs = np.clip(np.arange(x0 - 1, x0 + 3), 0, W - 1)
            ys = np.clip(np.arange(y0 - 1, y0 + 3), 0, H - 1)
            fp = val[np.ix_(ys, xs)].reshape(-1, 4)
            assert np.all(r[y, x] >= fp.min(0) - 1e-6) and np.all(r[y, x] <= fp.max(0) + 1e-6)
            same += np.allclose(r[y, x], ex[y, x], atol=1e-12)
    assert same > 0


def test_box_and_mask_semantics_bicubic():
    """Box is exact iff the AABB area <= E*a (then evals = area); Mask-16 / -11 exact iff
    the AABB fits and n <= E*a; an exact Box or Mask wave is an exact List wave, and
    every exact wave equals the 16-tap filter."""
    W = H = 256
    tex = bc1_tex(W, H, 2, "image")
    for m, th in [(2.5, 10.0), (3.2, 40.0), (4.0, 0.0)]:
        uv, _ = synthetic.rotated_quad(64, 32, W, H, m, th)
        ref = filter_frame(tex, uv, None, M_4TAP, filter=FILTER_CATMULL_ROM, debug=False)["out"]
        lst = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_C, filter=FILTER_CATMULL_ROM,
                                         max_evals=2, debug=False)["rec"])
        for mode in (M_BOX, M_MASK16, M_MASK11):
            r = filter_frame(tex, uv, None, mode, FB_C, filter=FILTER_CATMULL_ROM, max_evals=2, debug=False)
            d = decode_record(r["rec"])
            ex = d["path"] == 0
            assert np.all(lst["path"][ex] == 0)
            assert np.all(d["evals"][ex] <= 2 * d["a"][ex])
            px = np.repeat(np.repeat(ex, 4, 0), 8, 1)
            np.testing.assert_allclose(r["out"][px], ref[px], atol=1e-12)
        assert (d["path"] == 0).any()
