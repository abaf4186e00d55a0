"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage (P:n = PAPER.md line) or the closed form it checks.
None compares the oracle with itself or with the CUDA path.
"""
import numpy as np
import pytest

import oracle
import synthetic
from oracle.oracle import (FB_C, FB_CPLUS, FB_STF, FB_WC, FL_FORCE_FALLBACK, M_4TAP, M_COLLAB, M_STF,
                           M_WC, decode_record, filter_frame)
from tests.helpers import blocks_from, codes_word, golden_rows, ramp_texture, bc1_tex, mlp_tex

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ---------------------------------------------------------------- RNG (R-11) --
def test_philox_known_answers():
    """Random123 published KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    for row in golden_rows("philox4x32_10_kat.txt"):
        vals = [int(x, 16) for x in row]
        got = oracle.philox4x32_10(vals[0:4], vals[4:6])
        assert got.tolist() == vals[6:10]


# ------------------------------------------------------ h, h^-1 --
def test_fig2_bijection():
    for op, arg, bits, res in golden_rows("fig2_bijection.txt"):
        mask = sum(1 << int(b) for b in bits.split(","))
        f = oracle.h if op == "h" else oracle.h_inv
        assert f(int(arg), mask) == int(res)


def test_h_roundtrip_random_masks():
    """h^-1(h(i,B),B) = i for every set-bit rank (the bijection of P:395-412)."""
    rng = np.random.default_rng(0)
    for B in rng.integers(1, 1 << 32, 300, dtype=np.uint64):
        B = int(B)
        n = bin(B).count("1")
        for i in range(n):
            t = oracle.h(i, B)
            assert (B >> t) & 1
            assert oracle.h_inv(t, B) == i


# ------------------------------------------------------------ Eq. 2 --
def test_eq2_paper_statements():
    for n, c, l in golden_rows("eq2_spread.txt"):
        assert oracle.eq2(int(c), int(n)) == int(l)


def test_eq2_exhaustive_properties():
    """For every n in [0,30]: outputs distinct, in [0,31], include lanes 0 and 31,
    and equal round-half-up of 31(c-n)/(31-n) evaluated in exact rational arithmetic."""
    from fractions import Fraction
    for n in range(0, 31):
        ls = [oracle.eq2(c, n) for c in range(n, 32)]
        assert len(set(ls)) == len(ls)
        assert min(ls) == 0 and max(ls) == 31
        for c, l in zip(range(n, 32), ls):
            q = Fraction(31 * (c - n), 31 - n)
            assert l == int(q + Fraction(1, 2)) if q.denominator != 1 else l == q


# ------------------------------------------------- footprint --
def test_footprint_texel_center_and_clamp():
    W = H = 16
    # uv*dims - 0.5 = (3, 5): upper-left (3,5), st = (0,0)
    ids, st = oracle.footprint(3.5 / W, 5.5 / H, W, H)
    assert ids.tolist() == [5 * W + 3, 5 * W + 4, 6 * W + 3, 6 * W + 4]
    assert st.tolist() == [0.0, 0.0]
    # st = (1/2, 1/2) exactly
    ids, st = oracle.footprint(4.0 / W, 6.0 / H, W, H)
    assert st.tolist() == [0.5, 0.5] and ids[0] == 5 * W + 3
    # uv = 1: x0 = W-1, x0+1 clamps to W-1 (clamp-to-edge, R-2 i)
    ids, st = oracle.footprint(1.0, 1.0, W, H)
    assert ids.tolist() == [W * W - 1] * 4
    # uv = 0: x0 = -1 clamps to 0, x0+1 = 0
    ids, st = oracle.footprint(0.0, 0.0, W, H)
    assert ids.tolist() == [0, 0, 0, 0] and st.tolist() == [0.5, 0.5]


# -------------------------------------------------------- BC1 decode (R-9) --
def test_bc1_hand_vectors():
    for c0, c1, code, r, g, b, a in golden_rows("bc1_hand_vectors.txt"):
        word = codes_word([[int(code)] * 4] * 4)
        blk = blocks_from(np.array([int(c0, 16)]), np.array([int(c1, 16)]), np.array([word]))
        for (x, y) in [(0, 0), (3, 1), (2, 3)]:
            assert oracle.bc1_texel(blk, 4, x, y).tolist() == [int(r), int(g), int(b), int(a)]


def test_bc1_index_addressing():
    """Texel (x,y) reads index bits 2*(4(y&3)+(x&3)) of block ((y>>2)*(W>>2)+(x>>2))."""
    rng = np.random.default_rng(5)
    W, H = 16, 8
    nb = (W // 4) * (H // 4)
    c0 = np.full(nb, 0xF800)
    c1 = np.full(nb, 0x001F)
    codes = rng.integers(0, 4, (nb, 4, 4))
    idx = np.array([codes_word(c) for c in codes])
    blk = blocks_from(c0, c1, idx)
    red = {0: 255, 1: 0, 2: 170, 3: 85}
    for y in range(H):
        for x in range(W):
            bi = (y // 4) * (W // 4) + x // 4
            assert oracle.bc1_texel(blk, W, x, y)[0] == red[int(codes[bi, y % 4, x % 4])]


# ----------------------------- exact path = bilinear: linear-ramp closed form --
@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("mode", [M_4TAP, M_COLLAB])
def test_linear_ramp_closed_form(axis, mode):
    """Bilinear interpolation reproduces a linear function exactly: for G8(k) = 4k the
    filtered green is 4*clamp(f, 0, 15)/255 with f = uv*W - 0.5 (fp32 R-2),
    for every magnified wave that the method resolves exactly."""
    tex, W, H = ramp_texture(axis, height=16)
    rng = np.random.default_rng(1)
    wf, hf = 40, 20
    uv = np.empty((hf, wf, 2), np.float32)
    # smooth, magnified mapping (m ~ 3-4) plus a few off-texture pixels to hit the clamp
    py, px = np.mgrid[0:hf, 0:wf].astype(np.float64)
    uv[..., 0] = (px * 0.29 + py * 0.07) / W - 0.1 + rng.random() * 0.01
    uv[..., 1] = (py * 0.27 - px * 0.05) / H + 0.05
    r = filter_frame(tex, uv, None, mode, FB_STF)
    d = decode_record(r["rec"])
    coord = uv[..., 0] if axis == "x" else uv[..., 1]
    dim = np.float32(W if axis == "x" else H)
    f = (coord.astype(np.float32) * dim) - np.float32(0.5)
    expect = 4.0 * np.clip(f.astype(np.float64), 0.0, 15.0) / 255.0
    exact_px = np.repeat(np.repeat(d["path"] == (0 if mode == M_COLLAB else 5), 4, 0), 8, 1)[:hf, :wf]
    assert exact_px.mean() > 0.9
    g = r["out"][..., 1]
    np.testing.assert_allclose(g[exact_px], expect[exact_px], atol=1e-12)
    assert np.all(r["out"][..., 0][exact_px] == 0.0) and np.all(r["out"][..., 3][exact_px] == 1.0)


# -------------------------------------------------- constant texture invariants --
@pytest.mark.parametrize("mode,fb,flags", [(M_4TAP, 0, 0), (M_STF, 0, 0), (M_WC, 0, 0),
                                           (M_COLLAB, FB_STF, FL_FORCE_FALLBACK),
                                           (M_COLLAB, FB_WC, FL_FORCE_FALLBACK),
                                           (M_COLLAB, FB_C, FL_FORCE_FALLBACK),
                                           (M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK),
                                           (M_COLLAB, FB_CPLUS, 0)])
def test_constant_texture_gives_constant(mode, fb, flags):
    """Partition of unity and Eq. 1's weights (w + (1 - Sum w) = 1) make
    every estimator return the constant; uncovered pixels return 0 (DESIGN.md boundary)."""
    tex = bc1_tex(64, 64, 3, "constant")
    uv, g = synthetic.rotated_quad(37, 21, 64, 64, 1.3, 33.0, coverage="circle", radius=9.0)
    r = filter_frame(tex, uv, g, mode, fb, flags, seed=9)
    cov = ~np.isnan(uv[..., 0])
    c = r["out"][cov]
    np.testing.assert_allclose(c, np.broadcast_to(c[0], c.shape), atol=1e-12)
    assert np.all(r["out"][~cov] == 0.0)


# -------------------------------------------- unique set = brute force set size --
def test_unique_count_brute_force():
    """n in the wave record equals |set of footprint ids| over active lanes (List semantics,
    P:300-321), computed here with a Python set on tiny random frames."""
    rng = np.random.default_rng(7)
    W = H = 32
    tex = bc1_tex(W, H, 1, "random")
    for trial in range(4):
        wf, hf = 19, 9
        uv = rng.random((hf, wf, 2)).astype(np.float32) * (0.3 if trial % 2 else 1.0)
        uv[rng.random((hf, wf)) < 0.2, 0] = np.nan
        r = filter_frame(tex, uv, None, M_COLLAB, FB_C, seed=trial)
        d = decode_record(r["rec"])
        for wy in range(d["n"].shape[0]):
            for wx in range(d["n"].shape[1]):
                ids = set()
                a = 0
                for ly in range(4):
                    for lx in range(8):
                        x, y = wx * 8 + lx, wy * 4 + ly
                        if x < wf and y < hf and not np.isnan(uv[y, x, 0]):
                            a += 1
                            fid, _ = oracle.footprint(float(uv[y, x, 0]), float(uv[y, x, 1]), W, H)
                            ids.update(int(i) for i in fid)
                assert d["a"][wy, wx] == a
                assert d["n"][wy, wx] == len(ids)
                assert d["path"][wy, wx] == (0 if len(ids) <= a else 3)


# ------------------------------------------------------ the 54 bound --
def test_54_texel_bound_at_unit_magnification():
    rows = {r[0]: r[1:] for r in golden_rows("thresholds.txt")}
    tex = bc1_tex(1024, 1024, 1, "constant")
    best = {}
    for th in range(0, 91, 1):
        uv, _ = synthetic.rotated_quad(256, 256, 1024, 1024, 1.0, float(th))
        n = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_STF, debug=False)["rec"])["n"]
        best[th] = int(n.max())
    assert max(best.values()) == int(rows["bound_m1_max"][0])
    assert best[30] == int(rows["bound_m1_at30"][0])


# ----------------------------------------------- perfect above 1.59 --
@pytest.mark.slow
def test_perfect_filtering_threshold():
    rows = {r[0]: r[1:] for r in golden_rows("thresholds.txt")}
    tex = bc1_tex(1024, 1024, 1, "constant")
    m_ok = float(rows["perfect_above"][0])
    for th in np.arange(0.0, 90.01, 2.5):
        for j in range(2):
            uv, _ = synthetic.rotated_quad(640, 640, 1024, 1024, m_ok, float(th), jitter_seed=j)
            n = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_STF, debug=False)["rec"])["n"]
            assert n.max() <= 32, (th, j)
    m_bad, th_bad = float(rows["fails_at"][0]), float(rows["fails_at"][1])
    worst = 0
    for j in range(6):
        uv, _ = synthetic.rotated_quad(800, 800, 1024, 1024, m_bad, th_bad, jitter_seed=j)
        worst = max(worst, int(decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_STF, debug=False)["rec"])["n"].max()))
    assert worst > 32


# ---------------------------------------------- edge remapping --
def test_edge_remap_example():
    """Active mask 11101010 (lanes {1,3,5,6,7}) needing 4 texels still succeeds;
    rank r is produced by lane h(r, A)."""
    W = H = 16
    tex = bc1_tex(W, H, 2, "image")
    uv = np.full((4, 8, 2), np.nan, np.float32)
    lanes = [1, 3, 5, 6, 7]
    for l in lanes:
        uv[l // 8, l % 8] = (5.3 / W, 7.6 / H)    # all share one 2x2 footprint: n = 4
    r = filter_frame(tex, uv, None, M_COLLAB, FB_STF)
    d = decode_record(r["rec"])
    assert (d["n"][0, 0], d["a"][0, 0], d["path"][0, 0], d["evals"][0, 0]) == (4, 5, 0, 4)
    fid, _ = oracle.footprint(5.3 / W, 7.6 / H, W, H)
    U = sorted(set(int(i) for i in fid))
    pid = r["produced_id"].reshape(-1)
    assert [int(pid[l]) for l in lanes[:4]] == U and pid[7] == 0xFFFFFFFF
    r4 = filter_frame(tex, uv, None, M_4TAP)
    np.testing.assert_array_equal(r["out"], r4["out"])


def test_clamp_duplicates_single_lane_needs_fallback():
    """'two texels are needed (e.g., due to clamping), but there is only a single active lane'
    -> fallback; a lane in the texture corner needs 1 texel -> exact."""
    W = H = 16
    tex = bc1_tex(W, H, 2, "image")
    uv = np.full((4, 8, 2), np.nan, np.float32)
    uv[2, 3] = (1.0, 7.6 / H)            # x clamped: 2 distinct texels
    d = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_C)["rec"])
    assert (d["n"][0, 0], d["a"][0, 0], d["path"][0, 0]) == (2, 1, 3)
    uv[2, 3] = (1.0, 1.0)                # both clamped: 1 texel
    d = decode_record(filter_frame(tex, uv, None, M_COLLAB, FB_C)["rec"])
    assert (d["n"][0, 0], d["a"][0, 0], d["path"][0, 0]) == (1, 1, 0)


# --------------------------------------------------- fallbacks --
def _texel_values(tex, ids):
    W = tex["width"]
    return np.array([oracle.bc1_texel(tex["bc1"], W, int(i) % W, int(i) // W) / 255.0 for i in ids])


def test_fallback_estimator_special_cases_and_convexity():
    """Eq. 1: output is a convex combination of the known texels (weights
    w_i + (1 - Sum w)/N >= 0 summing to 1), N = 1 returns the one-tap value, and a lane
    whose whole footprint is known is exact."""
    W = H = 64
    tex = bc1_tex(W, H, 4, "random")
    uv, g = synthetic.rotated_quad(32, 16, W, H, 1.1, 27.0, jitter_seed=3)
    exact = filter_frame(tex, uv, g, M_4TAP)["out"]
    for fb in (FB_C, FB_CPLUS, FB_WC):
        r = filter_frame(tex, uv, g, M_COLLAB, fb, FL_FORCE_FALLBACK, seed=11)
        n_exact = 0
        for y in range(16):
            for x in range(32):
                wpid = r["produced_id"][(y // 4) * 4:(y // 4) * 4 + 4, (x // 8) * 8:(x // 8) * 8 + 8]
                pid = set(int(p) for p in wpid.reshape(-1) if p != 0xFFFFFFFF)
                ids, st = oracle.footprint(float(uv[y, x, 0]), float(uv[y, x, 1]), W, H)
                w = [(1 - st[0]) * (1 - st[1]), st[0] * (1 - st[1]), (1 - st[0]) * st[1], st[0] * st[1]]
                need = {int(i) for i, wi in zip(ids, w) if wi != 0}
                known = [i for i in need if i in pid]
                vals = _texel_values(tex, known)
                c = r["out"][y, x]
                assert len(known) >= 1
                assert np.all(c >= vals.min(0) - 1e-12) and np.all(c <= vals.max(0) + 1e-12)
                # the special cases are the values themselves, bit for bit: N = 1 returns the
                # one texel, an all-known footprint the exact bilinear result of
                # the 4TAP mode — not the general formula's rounding of them
                if len(known) == 1:
                    np.testing.assert_array_equal(c, vals[0])
                if len(known) == len(need):
                    np.testing.assert_array_equal(c, exact[y, x])
                    n_exact += 1
        assert n_exact > 0


def test_stf_expectation_is_bilinear():
    """One-tap STF picks a texel with probability equal to its weight, so its
    average over independent draws converges to the bilinear value."""
    W = H = 16
    tex = bc1_tex(W, H, 6, "random")
    uv = np.empty((32, 64, 2), np.float32)
    uv[..., 0], uv[..., 1] = 6.8 / W, 9.35 / H           # s = 0.3, t = 0.85 (approximately)
    ref = filter_frame(tex, uv[:1, :1], None, M_4TAP)["out"][0, 0]
    acc = np.zeros(4)
    nfr = 24
    for f in range(nfr):
        acc += filter_frame(tex, uv, None, M_STF, seed=123, frame_index=f, debug=False)["out"].mean((0, 1))
    acc /= nfr
    # 49152 draws: std of the mean <= 0.5/sqrt(49152) ~ 2.3e-3
    np.testing.assert_allclose(acc, ref, atol=1e-2)


def test_stf_picks_with_probability_exactly_the_weight():
    """One-tap STF picks the right texel column with probability s and the lower row with
    probability t ('probability based on its corresponding filter weight').  The
    uniforms lie on the 2^-24 grid (R-11), so P(pick right) = s holds exactly only for the
    event {u < s}: it has s * 2^24 grid points, {u <= s} one more.  A pixel whose s equals its
    own u0 exactly (constructed: uv.x = (1/2 + u0) / W with W = 16, exact in fp32) must keep
    the left column; t = u1 + 2^-24 must take the lower row.  Choosing u0 > u1 also fixes the
    stream convention of R-11 (u0 decides x, u1 decides y)."""
    W = H = 16
    tex = bc1_tex(W, H, 2, "random")
    found = 0
    for seed in range(1, 400):
        r = oracle.philox4x32_10([0, 0, 0, 0], [seed & 0xFFFFFFFF, 0])
        u0, u1 = (int(r[0]) >> 8) / 2.0 ** 24, (int(r[1]) >> 8) / 2.0 ** 24
        if not (u1 < u0 < 0.5 and u1 + 2.0 ** -24 < 0.5):
            continue
        uv = np.full((4, 8, 2), np.nan, np.float32)
        uv[0, 0] = (np.float32((0.5 + u0) / W), np.float32((0.5 + u1 + 2.0 ** -24) / H))
        ids, st = oracle.footprint(float(uv[0, 0, 0]), float(uv[0, 0, 1]), W, H)
        assert float(st[0]) == u0 and float(st[1]) == u1 + 2.0 ** -24   # the construction is exact
        sel = int(filter_frame(tex, uv, None, M_STF, seed=seed)["selection"][0, 0]) & 3
        assert sel == 2, (seed, u0, u1, sel)   # left column (u0 < s false), lower row (u1 < t)
        found += 1
        if found == 8:
            break
    assert found == 8


def test_cplus_extra_pick_probability_is_the_merged_weight_exactly():
    """A C+ spare lane picks an unplanned texel of its served lane with probability equal to
    its merged weight over the candidates' sum (R-18 v).  With u2 on the 2^-24 grid
    the first candidate's event {u2 * wsum < w_0} has exactly w_0 / wsum * 2^24 points only
    with a strict comparison, so at a constructed tie (w_0 = u2 * wsum exactly) the pick must
    be the second candidate.  Construction: lanes 0, 1, 2 share one footprint with t = 1/2 and
    s = 1 - u2(lane 2) (exact in fp32); every STF pick is in the lower row and both LL and LR
    are picked (n_p = 2), so lane 2 (active rank 2) serves lane 0 (Eq. 2 with n_p = a - 1)
    and its candidates are UL (weight (1 - s)/2 = u2/2) and UR (s/2), wsum = 1/2."""
    W = H = 16
    tex = bc1_tex(W, H, 2, "random")
    found = 0
    for seed in range(1, 3000):
        us = [oracle.philox4x32_10([x, 0, 0, 0], [seed, 0]) for x in range(3)]
        u = [[(int(r[k]) >> 8) / 2.0 ** 24 for k in range(3)] for r in us]
        s_ = 1.0 - u[2][2]
        if not (0.0 < s_ < 0.5) or any(ui[1] >= 0.5 for ui in u):
            continue
        picks = {(1 if ui[0] < s_ else 0) + 2 for ui in u}
        if picks != {2, 3}:
            continue
        uv = np.full((4, 8, 2), np.nan, np.float32)
        uv[0, 0:3] = (np.float32((0.5 + s_) / W), np.float32((0.5 + 0.5) / H))
        ids, st = oracle.footprint(float(uv[0, 0, 0]), float(uv[0, 0, 1]), W, H)
        assert float(st[0]) == s_ and float(st[1]) == 0.5   # the construction is exact
        r = filter_frame(tex, uv, None, M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK, seed=seed)
        assert (int(r["selection"][0, 2]) >> 8) & 31 == 0 and int(r["selection"][0, 2]) & (1 << 5)
        assert int(r["produced_id"][0, 2]) == int(ids[1]), (seed, s_)   # UR, not UL
        found += 1
        if found == 6:
            break
    assert found == 6


def test_cplus_plan_and_spread():
    """C+ (P:485-518): planned texels produced exactly once by the first n_p active lanes;
    spare lane of active rank j serves lane h(Eq.2(j), A); <= 1 evaluation per lane."""
    W = H = 256
    tex = bc1_tex(W, H, 8, "image")
    uv, g = synthetic.rotated_quad(64, 32, W, H, 1.4, 41.0, jitter_seed=1)
    r = filter_frame(tex, uv, g, M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK, seed=5)
    d = decode_record(r["rec"])
    for wy in range(8):
        for wx in range(8):
            sel = r["selection"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
            pid = r["produced_id"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
            lanes_uv = uv[wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1, 2)
            planned = []
            for l in range(32):
                ids, _ = oracle.footprint(float(lanes_uv[l, 0]), float(lanes_uv[l, 1]), W, H)
                planned.append(int(ids[sel[l] & 3]))
            P = sorted(set(planned))
            npl = len(P)
            assert pid[:npl].tolist() == P
            spares = [l for l in range(npl, 32)]
            for l in spares:
                assert (sel[l] >> 5) & 1
                assert (sel[l] >> 8) & 31 == oracle.eq2(l, npl)
                if (sel[l] >> 4) & 1:
                    assert pid[l] not in P
            produced = int((pid != 0xFFFFFFFF).sum())
            assert d["evals"][wy, wx] == produced <= 32
            assert d["path"][wy, wx] == 4


def test_fallback_quality_ordering():
    """P:1683-1684 (Fig. 12, fallback for every pixel): C beats one-tap STF, and C+ beats C,
    with C+ improving as magnification grows (spare lanes). PSNR vs bilinear."""
    tex = bc1_tex(256, 256, 3, "image")
    psnr = {}
    for m in (1.2, 2.0):
        mse = {}
        for fb in (FB_STF, FB_WC, FB_C, FB_CPLUS):
            e = 0.0
            for th, s in [(10.0, 0), (30.0, 1), (45.0, 2)]:
                uv, g = synthetic.rotated_quad(96, 64, 256, 256, m, th, jitter_seed=s)
                ref = filter_frame(tex, uv, g, M_4TAP, debug=False)["out"]
                out = filter_frame(tex, uv, g, M_COLLAB, fb, FL_FORCE_FALLBACK, seed=s + 1, debug=False)["out"]
                e += float(((out - ref) ** 2).mean())
            mse[fb] = e / 3
        psnr[m] = {k: 10 * np.log10(1 / v) for k, v in mse.items()}
        assert psnr[m][FB_CPLUS] > psnr[m][FB_C] > psnr[m][FB_STF]
        assert psnr[m][FB_WC] > psnr[m][FB_STF]
    assert psnr[2.0][FB_CPLUS] > psnr[1.2][FB_CPLUS] + 3.0


# ------------------------------------------------------- records and modes --
def test_record_fields_by_mode():
    """evals: 4TAP = 4a, STF/WC = a; n = 0xFF outside COLLAB; magnified class
    (R-20) from an analytic Jacobian: m = 1.25 -> magnified, m = 0.8 -> not."""
    tex = bc1_tex(128, 128, 1, "image")
    for m, mag in [(1.25, 1), (0.8, 0)]:
        uv, g = synthetic.rotated_quad(29, 10, 128, 128, m, 20.0)
        for mode, path in [(M_4TAP, 5), (M_STF, 6), (M_WC, 7)]:
            d = decode_record(filter_frame(tex, uv, g, mode, seed=1)["rec"])
            assert np.all(d["n"] == 0xFF) and np.all(d["path"] == path)
            assert np.all(d["evals"] == (4 if mode == M_4TAP else 1) * d["a"])
            assert np.all(d["magnified"] == mag)
            assert d["partial"].tolist() == [[0, 0, 0, 1]] * 2 + [[1, 1, 1, 1]]


# --------------------------------------------- latent-MLP decode (R-10) --
def test_mlp_decode_matches_independent_fp64():
    """Our synthetic NTC-style format (parity unpinned by the paper): the oracle's decode
    equals an independent numpy fp64 forward pass of the stated definition."""
    W = H = 32
    t = mlp_tex(W, H, 4)
    lat = t["latent"].astype(np.float64)
    p = t["mlp"].astype(np.float64)
    W1 = p[:384].reshape(32, 12); b1 = p[384:416]; W2 = p[416:1440].reshape(32, 32); b2 = p[1440:1472]
    W3 = p[1472:1600].reshape(4, 32); b3 = p[1600:1604]
    for (x, y) in [(0, 0), (5, 9), (31, 31), (17, 2)]:
        gx, gy = (x - 1.5) / 4, (y - 1.5) / 4
        x0, y0 = int(np.floor(gx)), int(np.floor(gy))
        fx, fy = gx - x0, gy - y0
        cl = lambda v, n: min(max(v, 0), n - 1)
        z = ((1 - fx) * (1 - fy) * lat[cl(y0, 8), cl(x0, 8)] + fx * (1 - fy) * lat[cl(y0, 8), cl(x0 + 1, 8)]
             + (1 - fx) * fy * lat[cl(y0 + 1, 8), cl(x0, 8)] + fx * fy * lat[cl(y0 + 1, 8), cl(x0 + 1, 8)])
        feat = np.concatenate([z, [((x & 3) - 1.5) / 2, ((y & 3) - 1.5) / 2, ((x >> 2) & 1) - 0.5, ((y >> 2) & 1) - 0.5]])
        h1 = np.maximum(W1 @ feat + b1, 0)
        h2 = np.maximum(W2 @ h1 + b2, 0)
        o = np.clip(W3 @ h2 + b3, 0, 1)
        np.testing.assert_allclose(oracle.mlp_texel(t["latent"], t["mlp"], W, H, x, y), o, atol=1e-12)


# ------------------------------------------- Box / Mask sampling (Fig. 4) --
@pytest.mark.slow
def test_box_threshold_45_degrees():
    """Box needs m > 2.35 at 45°; at m = 2.36 it is perfect for every rotation."""
    rows = {r[0]: r[1:] for r in golden_rows("thresholds.txt")}
    tex = bc1_tex(1024, 1024, 1, "constant")
    m_bad, th_bad = float(rows["box_fails_at"][0]), float(rows["box_fails_at"][1])
    fails = 0
    for j in range(6):
        uv, _ = synthetic.rotated_quad(800, 800, 1024, 1024, m_bad, th_bad, jitter_seed=j)
        fails += int((decode_record(filter_frame(tex, uv, None, 4, FB_STF, debug=False)["rec"])["path"] != 0).sum())
    assert fails > 0
    m_ok = float(rows["box_perfect_above"][0])
    for th in np.arange(0.0, 90.01, 5.0):
        uv, _ = synthetic.rotated_quad(640, 640, 1024, 1024, m_ok, float(th), jitter_seed=1)
        assert np.all(decode_record(filter_frame(tex, uv, None, 4, FB_STF, debug=False)["rec"])["path"] == 0), th


def test_mask_equals_list_and_11_equals_16_on_the_quad():
    """List and Mask 'cover identical areas' and the 11x11 mask gives results
    identical to 16x16 for bilinear: on rotated quads the records and images agree."""
    tex = bc1_tex(256, 256, 5, "image")
    for m, th in [(1.6, 37.5), (1.2, 20.0), (2.2, 45.0), (0.9, 10.0)]:
        uv, g = synthetic.rotated_quad(96, 48, 256, 256, m, th, jitter_seed=2)
        r = {mode: filter_frame(tex, uv, g, mode, FB_CPLUS, seed=3) for mode in (3, 5, 6)}
        for mode in (5, 6):
            np.testing.assert_array_equal(r[mode]["rec"], r[3]["rec"])
            np.testing.assert_array_equal(r[mode]["out"], r[3]["out"])


def test_box_produces_whole_aabb_and_is_exact():
    """Box: lane h(i,A) produces AABB texel (i mod w, i div w) (LaneIdxToCoord);
    evals = AABB area >= n; the image equals bilinear wherever it succeeds."""
    W = 64
    tex = bc1_tex(W, W, 9, "image")
    uv, g = synthetic.rotated_quad(40, 20, W, W, 3.0, 30.0, coverage="circle", radius=9.0)
    rb = filter_frame(tex, uv, g, 4, FB_C)
    r4 = filter_frame(tex, uv, g, 0, 0)
    d = decode_record(rb["rec"])
    ex = (d["path"] == 0) & (d["a"] > 0)
    assert ex.any() and np.all(d["evals"][ex] >= d["n"][ex])
    px = np.repeat(np.repeat(ex, 4, 0), 8, 1)[:20, :40]
    np.testing.assert_array_equal(rb["out"][px], r4["out"][px])
    # one wave in detail: produced ids are the AABB in row-major order on the active lanes
    wy, wx = np.argwhere(ex)[0]
    pid = rb["produced_id"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
    lanes_uv = uv[wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1, 2)
    act = [l for l in range(32) if not np.isnan(lanes_uv[l, 0])]
    xs, ys = [], []
    for l in act:
        ids, _ = oracle.footprint(float(lanes_uv[l, 0]), float(lanes_uv[l, 1]), W, W)
        xs += [int(i) % W for i in ids]
        ys += [int(i) // W for i in ids]
    bw = max(xs) - min(xs) + 1
    area = bw * (max(ys) - min(ys) + 1)
    expect = [(min(ys) + i // bw) * W + min(xs) + i % bw for i in range(area)]
    assert [int(pid[l]) for l in act[:area]] == expect


# ------------------------- Eq. 1's general case vs the WC renormalisation --
# P:477 reads Eq. 1's second term as estimating "the missing texel values as an unweighted
# average of the known ones".  So when every unknown footprint texel EQUALS the unweighted
# mean of the known ones, Eq. 1 reproduces exact bilinear — whatever the known set is — and a
# weight-renormalising estimator (Sum w p / Sum w) does not.  Conversely the renormalisation is
# exact when the unknown texels equal the WEIGHTED mean of the known ones (our WC reading,
# R-16), and Eq. 1 is not.  The footprint lies in one BC1 block whose 4-colour palette
# (c0 = pure red, c1 = pure blue) gives red/blue = code0 (255, 0), code1 (0, 255),
# code2 (170, 85), code3 (85, 170) — hand-decoded from R-9.
_PAL = {0: (255, 0), 1: (0, 255), 2: (170, 85), 3: (85, 170)}


def _one_block_texture(codes_at):
    """16x16 BC1 texture; block (0,0) has c0 = 0xF800 (red), c1 = 0x001F (blue) and the given
    codes at texel (x, y) (code 0 elsewhere); every other block is code 0."""
    W = H = 16
    codes = [[0] * 4 for _ in range(4)]
    for (x, y), c in codes_at.items():
        codes[y][x] = c
    nb = (W // 4) * (H // 4)
    c0 = np.full(nb, 0xF800)
    c1 = np.full(nb, 0x001F)
    idx = np.zeros(nb, np.uint32)
    idx[0] = codes_word(codes)
    return {"format": 1, "width": W, "height": H, "bc1": blocks_from(c0, c1, idx)}, W, H


def _probe_wave(W, H, s, t):
    """Lane 0 at fractional position (1 + s, 1 + t) in texel space (footprint = texels (1,1),
    (2,1), (1,2), (2,2), all weights nonzero); lanes 1 and 2 at the CENTRES of texels (1,1)
    and (2,1): with s = t = 0 their STF draw is the upper-left corner for every uniform (the
    strict u < s test, R-12), so they deterministically produce the upper row of lane 0's
    footprint; lane 0's own STF draw is random (any corner); the other 29 lanes are uncovered."""
    uv = np.full((4, 8, 2), np.nan, np.float32)
    uv[0, 0] = ((1.5 + s) / W, (1.5 + t) / H)
    uv[0, 1] = (1.5 / W, 1.5 / H)
    uv[0, 2] = (2.5 / W, 1.5 / H)
    return uv


def _bilinear_red_blue(codes, s, t):
    """Plain bilinear of the four hand-decoded palette values (UL, UR, LL, LR)."""
    w = [(1 - s) * (1 - t), s * (1 - t), (1 - s) * t, s * t]
    return np.array([sum(wk * _PAL[c][ch] for wk, c in zip(w, codes)) / 255.0 for ch in (0, 1)])


@pytest.mark.parametrize("fb", [FB_C, FB_CPLUS])
def test_eq1_unknown_equal_to_unweighted_mean_gives_bilinear(fb):
    """UL = code0 (255, 0), UR = code3 (85, 170), LL = LR = code2 (170, 85).  If lane 0 draws
    the upper row, K = {UL, UR} and both unknowns equal mean(K) = (170, 85); if it draws LL or
    LR, K = {UL, UR, code2} and the unknown one equals mean(K) = (170, 85) again.  Eq. 1 must
    then give exact bilinear in every case; the WC renormalisation must not."""
    codes = (0, 3, 2, 2)
    tex, W, H = _one_block_texture({(1, 1): 0, (2, 1): 3, (1, 2): 2, (2, 2): 2})
    s, t = 0.3, 0.6
    uv = _probe_wave(W, H, s, t)
    s32, t32 = (np.float32(uv[0, 0, 0]) * np.float32(W) - np.float32(0.5)) - 1, \
               (np.float32(uv[0, 0, 1]) * np.float32(H) - np.float32(0.5)) - 1
    expect = _bilinear_red_blue(codes, float(s32), float(t32))
    wc_off = 0
    for seed in range(12):
        r = filter_frame(tex, uv, None, M_COLLAB, fb, FL_FORCE_FALLBACK, seed=seed)
        assert decode_record(r["rec"])["path"][0, 0] == (3 if fb == FB_C else 4)
        got = r["out"][0, 0]
        np.testing.assert_allclose(got[[0, 2]], expect, atol=1e-12)
        np.testing.assert_allclose(got[[1, 3]], [0.0, 1.0], atol=1e-12)
        wc = filter_frame(tex, uv, None, M_COLLAB, FB_WC, FL_FORCE_FALLBACK, seed=seed)["out"][0, 0]
        wc_off += int(np.abs(wc[[0, 2]] - expect).max() > 1e-3)
    assert wc_off == 12


def test_wc_unknown_equal_to_weighted_mean_gives_bilinear():
    """UL = code0 (255, 0), UR = code1 (0, 255), LL = LR = code2 (170, 85), s = 1/3: the
    weighted mean of the upper row (1 - s)UL + sUR = (170, 85) equals the unknowns, so the
    renormalisation Sum w p / Sum w (R-16) reproduces bilinear for any known set containing
    the upper row; Eq. 1 (unweighted mean) does not."""
    codes = (0, 1, 2, 2)
    tex, W, H = _one_block_texture({(1, 1): 0, (2, 1): 1, (1, 2): 2, (2, 2): 2})
    uv = _probe_wave(W, H, 1.0 / 3.0, 0.55)
    s32 = float((np.float32(uv[0, 0, 0]) * np.float32(W) - np.float32(0.5)) - 1)
    t32 = float((np.float32(uv[0, 0, 1]) * np.float32(H) - np.float32(0.5)) - 1)
    expect = _bilinear_red_blue(codes, s32, t32)
    for seed in range(12):
        wc = filter_frame(tex, uv, None, M_COLLAB, FB_WC, FL_FORCE_FALLBACK, seed=seed)["out"][0, 0]
        np.testing.assert_allclose(wc[[0, 2]], expect, atol=1e-6)
        c = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=seed)["out"][0, 0]
        assert np.abs(c[[0, 2]] - expect).max() > 1e-3


def test_eq1_general_case_closed_form_on_random_known_sets():
    """Eq. 1 written out for one lane from the hand-decoded palette: the lane of _probe_wave on a
    texture where all four footprint texels differ; for every seed the result equals
    Sum_K w p + (1 - Sum_K w) mean_K(p) where K is read back as the set of produced ids (the
    estimator is a function of K only)."""
    codes = (0, 1, 3, 2)
    tex, W, H = _one_block_texture({(1, 1): 0, (2, 1): 1, (1, 2): 3, (2, 2): 2})
    uv = _probe_wave(W, H, 0.3, 0.6)
    s = float((np.float32(uv[0, 0, 0]) * np.float32(W) - np.float32(0.5)) - 1)
    t = float((np.float32(uv[0, 0, 1]) * np.float32(H) - np.float32(0.5)) - 1)
    w = [(1 - s) * (1 - t), s * (1 - t), (1 - s) * t, s * t]
    ids = [1 * W + 1, 1 * W + 2, 2 * W + 1, 2 * W + 2]
    seen = set()
    for seed in range(40):
        r = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=seed)
        prod = set(int(p) for p in r["produced_id"].reshape(-1) if p != 0xFFFFFFFF)
        K = [k for k in range(4) if ids[k] in prod]
        seen.add(tuple(K))
        if len(K) in (1, 4):
            continue
        Sw = sum(w[k] for k in K)
        for ch_i, ch in ((0, 0), (2, 1)):
            vals = [_PAL[codes[k]][ch] / 255.0 for k in K]
            e = sum(w[k] * v for k, v in zip(K, vals)) + (1 - Sw) * sum(vals) / len(K)
            assert abs(r["out"][0, 0, ch_i] - e) < 1e-12
    assert len(seen) >= 2     # the upper row plus at least one lower corner over the seeds


# --------------------------- R-20 magnified class on an anisotropic Jacobian --
@pytest.mark.parametrize("theta", [0.0, 25.0])
@pytest.mark.parametrize("cols,expect", [(((0.9, 0.3), (0.9, -0.3)), 1),    # |J_x|^2 = |J_y|^2 = 0.9
                                         (((0.9, 0.9), (0.3, -0.3)), 0)])   # |J_x|^2 = 1.62
def test_magnified_class_anisotropic(cols, expect, theta):
    """Magnification per screen axis: a wave is magnified iff one pixel step along screen x and
    along screen y each moves <= 1 texel (R-20).  The truth is taken by brute force from the uv
    buffer itself (finite differences of neighbouring pixels, independent of `grad`).  The two
    Jacobians are transposes of each other's classes: the row norms are (1.62, 0.18) where the
    column norms are (0.9, 0.9) and vice versa, so reading J transposed flips the class."""
    th = np.deg2rad(theta)
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    J = R @ np.array(cols, np.float64).T              # columns = screen-x / screen-y texel steps
    W = H = 256
    tex = bc1_tex(W, H, 2, "image")
    uv, g = synthetic.affine_quad(24, 8, W, H, J)
    du_x = (uv[:, 1:, :].astype(np.float64) - uv[:, :-1, :]) * (W, H)
    du_y = (uv[1:, :, :].astype(np.float64) - uv[:-1, :, :]) * (W, H)
    step2 = max(float((du_x ** 2).sum(-1).max()), float((du_y ** 2).sum(-1).max()))
    truth = int(step2 <= 1.0)
    assert truth == expect
    for mode in (M_COLLAB, M_4TAP):
        d = decode_record(filter_frame(tex, uv, g, mode, FB_C, seed=1)["rec"])
        assert np.all(d["magnified"] == truth)


# ----------------------------------- Eq. 2 on partial waves (R-18 iv) --
def test_eq2_partial_waves_exhaustive():
    """P:514-515's guarantees carried to a active lanes (a - 1 in place of 31): for every
    a in [1, 32] and n_p in [0, a - 1], the spare ranks c in [n_p, a - 1] map to DISTINCT
    served ranks in [0, a - 1], including 0 and a - 1 whenever a - n_p >= 2; a single spare
    rank maps to 0."""
    for a in range(1, 33):
        for n in range(0, a):
            ls = [oracle.eq2(c, n, a) for c in range(n, a)]
            assert all(0 <= l <= a - 1 for l in ls), (a, n, ls)
            assert len(set(ls)) == len(ls), (a, n, ls)
            if a - n >= 2:
                assert min(ls) == 0 and max(ls) == a - 1, (a, n, ls)
            else:
                assert ls == [0]


def test_cplus_spread_on_partial_waves():
    """C+ on a coverage-masked frame (circle): in every partial fallback wave the served lanes
    recorded in `selection` (b8-12) are active lanes, pairwise distinct, and include the first
    and last active lane whenever at least two lanes are spare (P:514-515 with edge remapping,
    P:1378-1380)."""
    W = H = 256
    tex = bc1_tex(W, H, 8, "image")
    uv, g = synthetic.rotated_quad(64, 32, W, H, 1.3, 33.0, coverage="circle", radius=14.0, jitter_seed=4)
    r = filter_frame(tex, uv, g, M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK, seed=3)
    d = decode_record(r["rec"])
    checked = 0
    for wy in range(d["a"].shape[0]):
        for wx in range(d["a"].shape[1]):
            a = int(d["a"][wy, wx])
            if a == 0 or a == 32:
                continue
            lanes_uv = uv[wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1, 2)
            act = [l for l in range(32) if not np.isnan(lanes_uv[l, 0])]
            sel = r["selection"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
            spare = [l for l in act if (sel[l] >> 5) & 1]
            served = [int((sel[l] >> 8) & 31) for l in spare]
            assert all(l in act for l in served)
            assert len(set(served)) == len(served)
            if len(spare) >= 2:
                assert act[0] in served and act[-1] in served
                checked += 1
    assert checked >= 5


def test_magnified_class_boundary_m_equals_one():
    """m = 1 (one texel per pixel, J = I or a rotation of it at 90°) is still magnification: the
    paper's magnification studies start at m = 1.0 (P:1632, P:1643 '[1.0, 2.5]'), and minified
    waves are those with a pixel BELOW 1.  fp16 1.0 and 0.0 are exact."""
    W = H = 128
    tex = bc1_tex(W, H, 2, "image")
    for J in ([[1.0, 0.0], [0.0, 1.0]], [[0.0, -1.0], [1.0, 0.0]]):
        uv, g = synthetic.affine_quad(16, 8, W, H, J)
        d = decode_record(filter_frame(tex, uv, g, M_COLLAB, FB_C, seed=1)["rec"])
        assert np.all(d["magnified"] == 1)
    uv, g = synthetic.affine_quad(16, 8, W, H, [[1.01, 0.0], [0.0, 1.0]])
    assert np.all(decode_record(filter_frame(tex, uv, g, M_COLLAB, FB_C, seed=1)["rec"])["magnified"] == 0)


def test_eq1_counts_only_nonzero_weight_texels():
    """the known set holds the unique texels 'with nonzero filter weights'.  Lane 0
    sits on a texel row (t = 0, s = 1/2: weights UL = UR = 1/2, LL = LR = 0); lanes 1 and 2
    (texel centres) produce UL and the zero-weight LL.  When lane 0 draws UL, its only known
    nonzero-weight texel is UL, so N = 1 and the result is exactly that texel —
    the known zero-weight LL must not enter N or the mean; when it draws UR, everything with
    nonzero weight is known and the result is exact bilinear."""
    tex, W, H = _one_block_texture({(1, 1): 0, (2, 1): 1, (1, 2): 3, (2, 2): 2})
    uv = np.full((4, 8, 2), np.nan, np.float32)
    uv[0, 0] = (2.0 / W, 1.5 / H)          # fx = 1.5, fy = 1.0: s = 1/2, t = 0
    uv[0, 1] = (1.5 / W, 1.5 / H)          # centre of (1,1) = UL
    uv[0, 2] = (1.5 / W, 2.5 / H)          # centre of (1,2) = LL (zero weight for lane 0)
    picks = set()
    for seed in range(16):
        r = filter_frame(tex, uv, None, M_COLLAB, FB_C, FL_FORCE_FALLBACK, seed=seed)
        corner = int(r["selection"][0, 0] & 3)
        picks.add(corner)
        got = r["out"][0, 0][[0, 2]] * 255.0
        if corner == 0:
            np.testing.assert_allclose(got, _PAL[0], atol=1e-9)
        else:
            assert corner == 1
            np.testing.assert_allclose(got, [0.5 * _PAL[0][c] + 0.5 * _PAL[1][c] for c in (0, 1)], atol=1e-9)
    assert picks == {0, 1}


def test_mask_grid_limits_on_a_16_wide_wave():
    """A full wave whose footprints tile a 16 x 2 texel strip (n = 32 = a): List and the 16 x 16
    mask resolve it exactly (the AABB fits the 16-wide grid), the 11 x 11 mask
    cannot (AABB wider than 11) and falls back."""
    W = H = 64
    tex = bc1_tex(W, H, 3, "image")
    uv = np.empty((4, 8, 2), np.float32)
    for lane in range(32):
        k = min(lane // 2, 14)             # footprint columns {k, k+1}, k = 0..14
        uv[lane // 8, lane % 8] = ((20 + k + 1.0) / W, (30 + 1.0) / H)   # fx = 20.5 + k, fy = 30.5
    expect = {M_COLLAB: 0, 5: 0, 6: 3}
    for mode, path in expect.items():
        d = decode_record(filter_frame(tex, uv, None, mode, FB_C, seed=1)["rec"])
        assert (d["n"][0, 0], d["a"][0, 0], d["path"][0, 0]) == (32, 32, path), mode


def test_cplus_extra_texels_come_from_the_served_lanes_footprint():
    """R-18 (i): a spare lane c serving lane l (Eq. 2) produces a texel of l's footprint with
    nonzero weight that is not planned (P:503-506 'its filter footprint ... spread out')."""
    W = H = 256
    tex = bc1_tex(W, H, 8, "image")
    uv, g = synthetic.rotated_quad(64, 32, W, H, 1.4, 41.0, jitter_seed=1)
    r = filter_frame(tex, uv, g, M_COLLAB, FB_CPLUS, FL_FORCE_FALLBACK, seed=5)
    n_extra = 0
    for wy in range(8):
        for wx in range(8):
            sel = r["selection"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
            pid = r["produced_id"][wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1)
            luv = uv[wy * 4:wy * 4 + 4, wx * 8:wx * 8 + 8].reshape(-1, 2)
            for c in range(32):
                if not ((sel[c] >> 4) & 1):
                    continue
                l = int((sel[c] >> 8) & 31)
                ids, st = oracle.footprint(float(luv[l, 0]), float(luv[l, 1]), W, H)
                w = [(1 - st[0]) * (1 - st[1]), st[0] * (1 - st[1]), (1 - st[0]) * st[1], st[0] * st[1]]
                assert int(pid[c]) in {int(i) for i, wi in zip(ids, w) if wi != 0}
                assert int(ids[(sel[c] >> 2) & 3]) == int(pid[c])
                n_extra += 1
    assert n_extra > 100
