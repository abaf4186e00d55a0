"""Pins of the CPU oracle, second batch (-m "not gpu"): the survivors of the round-2 mutation
run (scripts/oracle_mutants.py, profiles/r02/oracle_mutants.txt) each fail one of these.

Each test names the passage (P:n = PAPER.md line) or the DESIGN.md reading (R-n) it checks;
expected values come from the paper's rules, hand-decoded texels, exact rational arithmetic
or the Random123 generator (itself pinned by its published answers), never from the oracle's
own arithmetic on the same quantity.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synthetic
from oracle.oracle import (FB_C, FB_CPLUS, FL_FORCE_FALLBACK, M_COLLAB, M_STF, decode_record, filter_frame)
from tests.helpers import bc1_tex

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")
INVALID = 0xFFFFFFFF
M_MASK16, M_MASK11 = 5, 6


def test_cplus_spare_lanes_never_produce_zero_weight_texels():
    """P:466-468 ('the unique texels ... with nonzero filter weights') and P:503-506: a C+ spare
    lane draws only among its served lane's texels of nonzero weight.  Every lane samples a
    texel CENTRE (s = t = 0: weights (1, 0, 0, 0)), so its STF draw is its anchor for any
    uniform (R-12) and its only nonzero-weight texel is planned: the 16 spare lanes have no
    candidate and produce nothing.  The needed set still counts the zero-weight corners (R-4):
    16 columns x 4 rows = 64 > 32, so the wave falls back."""
    W = H = 64
    tex = bc1_tex(W, H, 4, "image")
    uv = np.empty((4, 8, 2), np.float32)
    for lane in range(32):
        lx, ly = lane % 8, lane // 8
        x, y = 8 + 2 * lx, 8 + 2 * (ly // 2)          # two rows of lanes share each anchor
        uv[ly, lx] = ((x + 0.5) / W, (y + 0.5) / H)   # exact in fp32: fx = x, fy = y
    r = filter_frame(tex, uv, None, M_COLLAB, FB_CPLUS, seed=3)
    d = decode_record(r["rec"])
    assert (d["n"][0, 0], d["a"][0, 0], d["path"][0, 0]) == (64, 32, 4)   # C+ fallback (path 4)
    assert d["evals"][0, 0] == 16                                           # n_p planned, no extras
    pid = r["produced_id"].reshape(-1)
    sel = r["selection"].reshape(-1)
    assert sorted(int(p) for p in pid if p != INVALID) == sorted(
        (8 + 2 * (ly // 2)) * W + 8 + 2 * lx for lx in range(8) for ly in (0, 2))
    spares = [c for c in range(32) if (sel[c] >> 5) & 1]
    assert len(spares) == 16 and all(pid[c] == INVALID and not (sel[c] >> 4) & 1 for c in spares)
    # every lane knows its only nonzero-weight texel: the colour is that texel (exact)
    for lane in range(32):
        lx, ly = lane % 8, lane // 8
        ref = oracle.bc1_texel(tex["bc1"], W, 8 + 2 * lx, 8 + 2 * (ly // 2)) / 255.0
        np.testing.assert_array_equal(r["out"][ly, lx], ref)


def test_eq1_one_known_texel_at_a_clamped_edge():
    """Eq. 1's N = 1 case (one known texel -> its value) where clamp-to-edge makes
    corners coincide (R-2, R-14: a texel's weight is the sum of its corners' weights).  Every
    lane samples the last texel column at s = 0 (u = (W - 1/2) / W, fx = W - 1: the right
    corners clamp onto the left ones with weight 0), so a lane's footprint is the two texels
    (W-1, y0) with weight 1 - t and (W-1, y0+1) with weight t, both nonzero.  Under the forced C
    fallback a lane that knows only one of them takes that texel's value; one that knows both is
    the exact blend."""
    W = H = 32
    tex = bc1_tex(W, H, 6, "random")
    rng = np.random.default_rng(11)
    uv = np.empty((4, 8, 2), np.float32)
    t = rng.uniform(0.05, 0.15, 32)                      # lanes mostly draw their upper texel
    rows = np.arange(32) % 8 * 2 + 8                     # y0: 4 lanes per row pair
    for lane in range(32):
        uv[lane // 8, lane % 8] = ((W - 0.5) / W, (rows[lane] + 0.5 + t[lane]) / H)
    r = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=9)
    known = {int(p) for p in r["produced_id"].reshape(-1) if p != INVALID}
    ones = 0
    for lane in range(32):
        ids, st = oracle.footprint(float(uv[lane // 8, lane % 8, 0]), float(uv[lane // 8, lane % 8, 1]), W, H)
        assert float(st[0]) == 0.0 and ids[0] == ids[1] and ids[2] == ids[3]
        up, lo = int(ids[0]), int(ids[2])
        pu = oracle.bc1_texel(tex["bc1"], W, up % W, up // W).astype(np.float64) / 255.0
        pl = oracle.bc1_texel(tex["bc1"], W, lo % W, lo // W).astype(np.float64) / 255.0
        got = r["out"][lane // 8, lane % 8]
        if up in known and lo in known:
            tt = float(st[1])
            np.testing.assert_allclose(got, (1 - tt) * pu + tt * pl, rtol=0, atol=1e-12)
        else:
            ones += 1
            np.testing.assert_array_equal(got, pu if up in known else pl)
    assert ones >= 8   # the construction exercises the N = 1 case


def test_partial_bit_for_one_uncovered_lane():
    """Record layout: bit 26 'partial' is set iff the wave has an
    inactive lane; a = popc(A).  One uncovered lane: a = 31, partial = 1."""
    W = H = 64
    tex = bc1_tex(W, H, 1, "image")
    uv = np.empty((4, 16, 2), np.float32)
    for y in range(4):
        for x in range(16):
            uv[y, x] = ((20.25 + 0.5 * x) / W, (20.25 + 0.5 * y) / H)
    uv[2, 11] = (np.nan, np.nan)                        # wave 1, lane 19
    d = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_C, seed=1)["rec"])
    assert (d["a"][0, 0], d["partial"][0, 0]) == (32, 0)
    assert (d["a"][0, 1], d["partial"][0, 1]) == (31, 1)


@pytest.mark.parametrize("k,exact11,exact16", [(9, True, True), (10, False, True), (14, False, True),
                                               (15, False, False)])
def test_mask_grid_width_limits(k, exact11, exact16):
    """Mask Sampling resolves a wave iff its texel AABB fits the mask (16 x 16, P:368-369;
    11 x 11) and n <= a; List has no AABB limit.  31 lanes sample the
    centre of texel (20, 30) (footprint columns 20-21), lane 0 the centre of (20 + k, 30)
    (columns 20+k .. 21+k): AABB width k + 2, n = 8."""
    W = H = 64
    tex = bc1_tex(W, H, 3, "image")
    uv = np.empty((4, 8, 2), np.float32)
    uv[:, :] = (20.5 / W, 30.5 / H)
    uv[0, 0] = ((20 + k + 0.5) / W, 30.5 / H)
    for mode, ok in ((M_COLLAB, True), (M_MASK16, exact16), (M_MASK11, exact11)):
        d = decode_record(filter_frame(tex, uv, None, mode, FB_C, seed=1)["rec"])
        assert d["n"][0, 0] == 8
        assert (d["path"][0, 0] == 0) == ok, (mode, k)


def _round_to_f32(x: Fraction) -> float:
    """x correctly rounded to binary32 (ties to even), by exact comparison of neighbours."""
    f = np.float32(float(x))
    cands = {f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))}
    def key(c):
        return (abs(Fraction(float(c)) - x), int(np.frombuffer(np.float32(c).tobytes(), np.uint32)[0]) & 1)
    return float(min(cands, key=key))


def test_footprint_position_is_one_rounding_of_u_times_w_minus_half():
    """R-2: fx = u*W - 1/2 rounded ONCE to fp32 (the listing's uv * txDim - 0.5, P:1109-1112,
    as a fused multiply-add).  Checked against exact rational arithmetic on widths that are not
    powers of two (where one and two roundings differ): x0 = floor(fx), s = fx - x0."""
    rng = np.random.default_rng(5)
    differ = 0
    for W in (12, 20, 100, 1000, 3000):
        us = np.concatenate([rng.uniform(1.0, 1.5, 300) / W, rng.uniform(0, 1, 300)]).astype(np.float32)
        for u in us:
            fx = _round_to_f32(Fraction(float(u)) * W - Fraction(1, 2))
            x0 = int(np.floor(fx))
            if not 0 <= x0 <= W - 2:
                continue
            ids, st = oracle.footprint(float(u), 0.5, W, 4)
            assert int(ids[0]) % W == x0 and float(st[0]) == fx - x0, (W, float(u))
            two = float(np.float32(np.float32(u) * np.float32(W)) - np.float32(0.5))
            differ += two != fx
    assert differ > 50   # the pin separates the two readings


@pytest.mark.parametrize("u,edge", [(-0.3, 0.0), (-1e-3, 0.0), (-16.0, 0.0), (1.0 + 1e-3, 1.0), (3.5, 1.0)])
def test_out_of_range_coordinates_clamp_to_the_edge(u, edge):
    """R-2 (clamp-to-edge addressing): a coordinate outside [0, 1] samples exactly
    as the nearest edge coordinate — same texel ids AND the same fractions s, t (so the same
    STF / C+ corner choices), on both axes."""
    W, H = 64, 32
    for v in (0.37, u):
        a = oracle.footprint(u, v, W, H)
        b = oracle.footprint(edge, v if v != u else edge, W, H)
        assert list(a[0]) == list(b[0]) and list(a[1]) == list(b[1]), (u, v)


def test_rng_counter_is_pixel_row_frame():
    """R-11: the uniforms of pixel (px, py) in frame f are Philox4x32-10 of counter
    (px, py, f, 0) under key (seed_lo, seed_hi) — the generator itself is pinned by the Random123
    answers (test_philox_known_answers).  Pixels sampling at s = t = 1/2 exactly reveal
    u0 < 1/2 and u1 < 1/2 (the top bits of r0, r1) through their STF corner (R-12)."""
    W = H = 64
    tex = bc1_tex(W, H, 2, "random")
    hf, wf = 8, 16
    uv = np.empty((hf, wf, 2), np.float32)
    for y in range(hf):
        for x in range(wf):
            uv[y, x] = ((x + 10 + 1.0) / W, (y + 20 + 1.0) / H)     # fx = x + 10.5: s = 1/2
    seed, frame = 0x9E3779B97F4A7C15, 5
    sel = filter_frame(tex, uv, None, M_STF, seed=seed, frame_index=frame)["selection"]
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for y in range(hf):
        for x in range(wf):
            r = oracle.philox4x32_10([x, y, frame, 0], key)
            k = int(r[0] < 2 ** 31) + 2 * int(r[1] < 2 ** 31)
            assert int(sel[y, x]) & 3 == k, (x, y)


@pytest.mark.parametrize("W,H", [(32, 8), (8, 32)])
def test_texel_addressing_on_non_square_textures(W, H):
    """id = y*W + x (R-3) and texel (x, y) lives in block (y>>2)*(W>>2) + (x>>2)
    (R-9): on a non-square texture, sampling the CENTRE of texel (x, y) (weights (1, 0, 0, 0))
    returns exactly that texel's decoded value, under 4-tap and under the collaborative path."""
    tex = bc1_tex(W, H, 12, "random")
    rng = np.random.default_rng(4)
    xs, ys = rng.integers(0, W - 1, 32), rng.integers(0, H - 1, 32)
    uv = np.empty((4, 8, 2), np.float32)
    for lane in range(32):
        uv[lane // 8, lane % 8] = ((xs[lane] + 0.5) / W, (ys[lane] + 0.5) / H)
    for mode in (0, M_COLLAB):
        out = filter_frame(tex, uv, None, mode, FB_C, seed=1)["out"]
        for lane in range(32):
            ref = oracle.bc1_texel(tex["bc1"], W, int(xs[lane]), int(ys[lane])).astype(np.float64) / 255.0
            np.testing.assert_array_equal(out[lane // 8, lane % 8], ref, err_msg=f"{mode} {lane}")


def test_positivized_stf_lobes_draw_independently():
    """R-27: the positivized STF baseline draws its positive-lobe tap with u0 and
    its negative-lobe tap with u1 — two independent draws, so over many pixels sampling the
    same point every (positive, negative) tap pair occurs.  With one shared uniform the pair
    would be a monotone function of it (at most n+ + n- - 1 = 15 of the 64 pairs).  Catmull-Rom
    at interior fractions: 8 positive and 8 negative taps.  The 4 x 4 footprint (texels 22..25
    on both axes) straddles four BC1 blocks 2 x 2 texels each, and each block gives its four
    texels the four distinct colours of 4-colour mode (codes 0..3), so all 16 tap values differ
    and each (positive, negative) pair has its own colour."""
    from tests.helpers import blocks_from, codes_word
    W = H = 64
    nb = (W // 4) * (H // 4)
    rng = np.random.default_rng(8)
    c0 = rng.integers(0x8000, 0xFFFF, nb)
    c1 = rng.integers(0x0000, 0x7FFF, nb)             # c0 > c1: 4-colour mode
    idx = np.zeros(nb, np.uint32)
    for by in (5, 6):
        for bx in (5, 6):
            codes = [[0] * 4 for _ in range(4)]
            xs = (2, 3) if bx == 5 else (0, 1)
            ys = (2, 3) if by == 5 else (0, 1)
            for k, (yy, xx) in enumerate((yy, xx) for yy in ys for xx in xs):
                codes[yy][xx] = k
            idx[by * (W // 4) + bx] = codes_word(codes)
    tex = {"format": 1, "width": W, "height": H, "bc1": blocks_from(c0, c1, idx)}
    hf, wf = 32, 64
    uv = np.empty((hf, wf, 2), np.float32)
    uv[:, :] = ((23 + 0.3 + 0.5) / W, (23 + 0.6 + 0.5) / H)   # x0 = y0 = 23, s ~ 0.3, t ~ 0.6
    out = filter_frame(tex, uv, None, M_STF, seed=17, filter=2)["out"].reshape(-1, 4)
    distinct = {tuple(np.round(c, 12)) for c in out}
    assert len(distinct) > 30, len(distinct)


def _cubic_pick_f32(w, u):
    """R-26's inverse-CDF tap choice in fp32 (first cumulative |w| > u * S, else the last
    nonzero tap) — the same decision the oracle and the kernels take in fp32."""
    S, last = np.float32(0), 0
    for i in range(4):
        S = np.float32(S + np.float32(abs(w[i])))
        if w[i] != 0:
            last = i
    target = np.float32(np.float32(u) * S)
    cum = np.float32(0)
    for i in range(4):
        cum = np.float32(cum + np.float32(abs(w[i])))
        if cum > target:
            return i
    return last


@pytest.mark.parametrize("filt", [1, 2])
def test_bicubic_eq1_at_a_clamped_edge_reproduces_the_filter(filt):
    """Eq. 1 estimates each unknown texel as the unweighted mean of the known ones, so
    it reproduces the full filter exactly when the unknown texels DO equal that mean.  At the
    left texture edge (x0 = 0: taps -1, 0 clamp onto column 0, R-24) the known-set weights are
    the merged sums of the coinciding taps (R-25); a wrong merge breaks the identity.
    Four lanes sample one point under the forced C fallback; their STF taps (R-26, drawn with
    the KAT-pinned Philox words of R-11) are the known set K.  The texture is then built so
    that K's texels average to the value M of every other texel (BC1 3-colour mode: black,
    colour e1 = 2M, and M = (c0 + c1) / 2, exact per channel)."""
    from tests.helpers import blocks_from
    W = H = 16
    u, v = (0.3 + 0.5) / W, (7.6 + 0.5) / H          # fx ~ 0.3 (x0 = 0), fy ~ 7.6 (interior)
    ids, st = oracle.footprint(u, v, W, H)
    assert int(ids[0]) % W == 0 and int(ids[0]) // W == 7
    from oracle.oracle import cubic_weights
    wx, wy = cubic_weights(filt, float(st[0])), cubic_weights(filt, float(st[1]))
    xs = [min(max(-1 + i, 0), W - 1) for i in range(4)]
    ys = [6 + j for j in range(4)]
    uv = np.full((4, 8, 2), np.nan, np.float32)
    uv[0, :4] = (u, v)
    for seed in range(1, 400):
        key = [seed, 0]
        K = set()
        for lane in range(4):
            r = oracle.philox4x32_10([lane, 0, 0, 0], key)
            i = _cubic_pick_f32(wx, (int(r[0]) >> 8) / 2.0 ** 24)
            j = _cubic_pick_f32(wy, (int(r[1]) >> 8) / 2.0 ** 24)
            K.add((xs[i], ys[j]))
        if len(K) >= 2 and any(x == 0 for x, _ in K) and len(K) < 12:
            break
    else:
        pytest.fail("no seed with a general Eq. 1 case on the merged column")
    nb = (W // 4) * (H // 4)
    codes = np.full((H, W), 2, np.int64)              # every texel M ...
    for k, (x, y) in enumerate(sorted(K)):            # ... but K: black / e1 alternating (M if odd)
        codes[y, x] = (k % 2) if not (len(K) % 2 and k == len(K) - 1) else 2
    idx = np.zeros(nb, np.uint32)
    for by in range(H // 4):
        for bx in range(W // 4):
            idx[by * (W // 4) + bx] = sum(int(codes[by * 4 + yy, bx * 4 + xx]) << (2 * (4 * yy + xx))
                                          for yy in range(4) for xx in range(4))
    tex = {"format": 1, "width": W, "height": H,
           "bc1": blocks_from(np.zeros(nb, np.int64), np.full(nb, 0xDD1B), idx)}   # c0 < c1: 3-colour mode
    full = filter_frame(tex, uv, None, 0, filter=filt)["out"][0, :4]
    eq1 = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=seed, filter=filt)["out"][0, :4]
    np.testing.assert_allclose(eq1, full, rtol=0, atol=2e-6)


# ------------------------------------------------ bicubic records / Box / C+ (R-24 .. R-28) --
def _taps(coord: float, dim: int):
    """R-24: fx = coord*dim - 1/2 (dim a power of two: exact), taps x0-1 .. x0+2 clamped, and
    the fractional position s."""
    fx = np.float32(np.clip(np.float32(coord), 0, 1) * np.float32(dim)) - np.float32(0.5)
    x0 = int(np.floor(fx))
    return [min(max(x0 - 1 + i, 0), dim - 1) for i in range(4)], float(fx - np.float32(x0))


def test_bicubic_full_filter_records_16_evaluations_per_pixel():
    """With a bicubic filter, BILINEAR_4TAP is the full 16-tap filter: 16 evaluations per active
    pixel (include/ctf.h; P:68-69's count for a 4 x 4 footprint), so a full wave's record holds
    512 — beyond the low 8 bits (bits 27-29 carry bits 8-10)."""
    W = H = 64
    tex = bc1_tex(W, H, 2, "image")
    uv = np.empty((8, 8, 2), np.float32)
    for y in range(8):
        for x in range(8):
            uv[y, x] = ((20.3 + 0.37 * x) / W, (20.6 + 0.41 * y) / H)
    uv[5, 3] = (np.nan, np.nan)
    d = decode_record(filter_frame(tex, uv, None, 0, filter=2)["rec"])
    assert (d["evals"][0, 0], d["a"][0, 0], d["path"][0, 0]) == (512, 32, 5)
    assert (d["evals"][1, 0], d["a"][1, 0]) == (16 * 31, 31)


def test_bicubic_box_with_two_evaluations_per_lane():
    """Box Sampling with max_evals = 2 (Fig. 13b): the wave is exact iff its texel
    AABB area is at most 2a, and then it evaluates the whole AABB.  A full wave at
    magnification 1.5 whose 4 x 4 footprints span an AABB of 33..64 texels: exact with E = 2,
    a fallback with E = 1."""
    W = H = 64
    tex = bc1_tex(W, H, 5, "image")
    uv = np.empty((4, 8, 2), np.float32)
    for y in range(4):
        for x in range(8):
            uv[y, x] = ((20.2 + (x + 0.5) / 1.5) / W, (24.7 + (y + 0.5) / 1.5) / H)
    xs = [t for v in uv[..., 0].ravel() for t in _taps(float(v), W)[0]]
    ys = [t for v in uv[..., 1].ravel() for t in _taps(float(v), H)[0]]
    area = (max(xs) - min(xs) + 1) * (max(ys) - min(ys) + 1)
    assert 32 < area <= 64, area
    for filt in (1, 2):
        d1 = decode_record(filter_frame(tex, uv, None, 4, FB_C, seed=3, filter=filt, max_evals=1)["rec"])
        d2 = decode_record(filter_frame(tex, uv, None, 4, FB_C, seed=3, filter=filt, max_evals=2)["rec"])
        assert d1["path"][0, 0] == 3                                    # fallback C
        assert (d2["path"][0, 0], d2["evals"][0, 0]) == (0, area)      # exact, the whole AABB


def test_bicubic_cplus_spares_at_texel_centres_produce_nothing():
    """Catmull-Rom interpolates: at a texel centre (s = t = 0) its weights are (0, 1, 0, 0) per
    axis, so the only nonzero-weight texel of a lane's 4 x 4 footprint is the sampled one, its
    STF draw (R-26) and its plan.  A C+ spare lane then has no candidate
    and produces nothing: evals = n_p.  (16 distinct anchors for 32 lanes; the needed set,
    zero-weight taps included, is 22 x 10 > 32 texels, so the wave falls back.)"""
    W = H = 64
    tex = bc1_tex(W, H, 4, "image")
    uv = np.empty((4, 8, 2), np.float32)
    for lane in range(32):
        lx, ly = lane % 8, lane // 8
        uv[ly, lx] = ((8 + 2 * lx + 0.5) / W, (8 + 2 * (ly // 2) + 0.5) / H)
    r = filter_frame(tex, uv, None, M_COLLAB, FB_CPLUS, seed=3, filter=2)
    d = decode_record(r["rec"])
    assert (d["a"][0, 0], d["path"][0, 0], d["evals"][0, 0]) == (32, 4, 16)
    pid, sel = r["produced_id"].reshape(-1), r["selection"].reshape(-1)
    spares = [c for c in range(32) if (sel[c] >> 5) & 1]
    assert len(spares) == 16 and all(pid[c] == INVALID and not (sel[c] >> 4) & 1 for c in spares)
    for lane in range(32):   # every lane's only nonzero-weight texel is known: the texel itself
        lx, ly = lane % 8, lane // 8
        ref = oracle.bc1_texel(tex["bc1"], W, 8 + 2 * lx, 8 + 2 * (ly // 2)).astype(np.float64) / 255.0
        np.testing.assert_allclose(r["out"][ly, lx], ref, rtol=0, atol=1e-12)


def test_bicubic_cplus_extras_follow_eq2_and_the_absolute_weights():
    """C+ with a bicubic filter (R-26 / R-28): spare lane c (active rank
    j >= n_p) serves lane l = h(Eq. 2(j), A) and draws an unplanned texel of l's 4 x 4 footprint
    with probability |w| / sum |w| — negative-lobe texels included.  Checked on full waves of a
    rotated quad away from the texture edges: the served lane, footprint membership with
    nonzero weight and not planned, the draw itself from the lane's u2 (the uniform R-11 gives
    the C+ extra pick), and the share of draws landing on negative-weight texels against its
    expectation (sum over draws of the candidates' negative |w| share)."""
    from oracle.oracle import cubic_weights
    W = H = 256
    tex = bc1_tex(W, H, 8, "image")
    uv, _ = synthetic.rotated_quad(128, 64, W, H, 1.2, 33.0, jitter_seed=2)
    r = filter_frame(tex, uv, None, M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK, seed=5, filter=2)
    neg, exp_neg, n_extra = 0, 0.0, 0
    for wy in range(16):
        for wx in range(16):
            sl = np.s_[wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8]
            pid, sel = r["produced_id"][sl].reshape(-1), r["selection"][sl].reshape(-1)
            luv = uv[sl].reshape(-1, 2)
            spare = [(sel[c] >> 5) & 1 for c in range(32)]
            n_p = 32 - sum(spare)
            assert spare == [0] * n_p + [1] * (32 - n_p)
            planned = {int(p) for p in pid[:n_p]}
            assert len(planned) == n_p and INVALID not in planned
            for c in range(n_p, 32):
                l = int((sel[c] >> 8) & 31)
                assert l == oracle.eq2(c, n_p, 32), (c, n_p, l)
                xs, s = _taps(float(luv[l, 0]), W)
                ys, t = _taps(float(luv[l, 1]), H)
                assert len(set(xs)) == 4 and len(set(ys)) == 4          # interior: no clamping
                wxs, wys = cubic_weights(2, s), cubic_weights(2, t)
                cells = {ys[j] * W + xs[i]: np.float32(wxs[i] * wys[j]) for j in range(4) for i in range(4)}
                cand = {k: abs(float(w)) for k, w in cells.items() if w != 0 and k not in planned}
                if not (sel[c] >> 4) & 1:
                    assert not cand and pid[c] == INVALID
                    continue
                assert int(pid[c]) in cand
                # the draw: inverse CDF of |w| over the candidates in row-major order, decided in
                # fp32 with the lane's third uniform u2 (R-11: r2 -> the C+ extra pick, R-18 v)
                px, py = wx * 8 + (c & 7), wy * 4 + (c >> 3)
                u2 = (int(oracle.philox4x32_10([px, py, 0, 0], [5, 0])[2]) >> 8) / 2.0 ** 24
                order = [ys[j] * W + xs[i] for j in range(4) for i in range(4) if ys[j] * W + xs[i] in cand]
                wsum = np.float32(0)
                for k in order:
                    wsum = np.float32(wsum + np.float32(cand[k]))
                target, cum, pick = np.float32(np.float32(u2) * wsum), np.float32(0), order[-1]
                for k in order:
                    cum = np.float32(cum + np.float32(cand[k]))
                    if cum > target:
                        pick = k
                        break
                assert int(pid[c]) == pick, (wx, wy, c)
                n_extra += 1
                neg += cells[int(pid[c])] < 0
                exp_neg += sum(w for k, w in cand.items() if cells[k] < 0) / sum(cand.values())
    assert n_extra > 500
    sd = np.sqrt(exp_neg)   # <= binomial sd
    print(f"extras {n_extra}, on negative-weight texels {neg} (expected {exp_neg:.1f})")
    assert neg > 0 and abs(neg - exp_neg) < 4 * sd + 5, (neg, exp_neg, n_extra)


def test_frame_stats_by_hand():
    """oracle.frame_stats (the expected ctf_stats) on hand-packed records
    (record layout of include/ctf.h): totals written out by hand."""
    def rec(evals, n, a, path, mag=0, partial=0):
        return (evals & 0xFF) | (n << 8) | (a << 16) | (path << 22) | (mag << 25) | (partial << 26) | ((evals >> 8) << 27)
    recs = np.array([rec(12, 12, 32, 0, mag=1),           # exact, magnified
                     rec(30, 45, 32, 4),                  # C+ fallback
                     rec(0, 0, 0, 0, partial=1),          # empty wave (not live)
                     rec(9, 9, 20, 0, mag=1, partial=1),  # partial exact wave
                     rec(512, 0xFF, 32, 5)], np.uint32)   # bicubic full filter
    st = oracle.frame_stats(recs)
    assert (st["waves_live"], st["waves_partial"], st["waves_exact"], st["waves_fallback"],
            st["waves_magnified"]) == (4, 1, 2, 1, 2)
    assert (st["pixels_active"], st["pixels_in_magnified_waves"]) == (116, 52)
    assert (st["texel_evals"], st["texel_evals_in_magnified_waves"]) == (563, 21)
    assert (st["max_unique_per_wave"], st["max_evals_per_lane"]) == (45, 16)
    assert {i: int(v) for i, v in enumerate(st["unique_hist"]) if v} == {9: 1, 12: 1, 45: 1}
    out = np.zeros((2, 2, 4)); ref = np.zeros((2, 2, 4))
    out[0, 1] = (0.5, 0.0, 0.0, 0.0); out[1, 0, 2] = -0.25
    st = oracle.frame_stats(recs, out, ref)
    assert (st["sum_sq_err"], st["max_abs_err"], st["err_pixels"]) == (0.3125, 0.5, 4)
