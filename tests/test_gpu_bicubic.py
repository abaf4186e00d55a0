"""GPU vs oracle parity for the bicubic filters (§5.4; R-24..R-28) — -m gpu.

Same bar as the bilinear parity tests: bit-exact per-wave records (n, evals, a, path,
magnified, partial), colours within 1e-5 per fp32 channel, through the C ABI.
"""
import numpy as np
import pytest

import synthetic
from tests.helpers import bc1_tex, mlp_tex

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ATOL = 1e-5
FILTERS = [1, 2]   # B-spline, Catmull-Rom
# (mode, fallback, flags, max_evals): full filter, positivized STF, List E=1/2 with every
# supported fallback (forced and natural), Box, Mask 16 / 11
MODES = [(0, 0, 0, 1), (1, 0, 0, 1),
         (3, 0, 0, 1), (3, 2, 0, 1), (3, 3, 0, 1), (3, 3, 0, 2), (3, 2, 0, 2),
         (3, 0, 2, 1), (3, 2, 2, 1), (3, 3, 2, 2),
         (4, 3, 0, 1), (4, 2, 0, 2), (5, 3, 0, 2), (6, 0, 0, 1), (6, 3, 0, 2)]


@pytest.fixture(scope="module")
def ctf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2506_17770_b200.ctf as c
    c.load_library()
    return c


def dev_tex(ctf, t):
    if t["format"] == 1:
        return ctf.Texture.bc1(t["bc1"], t["width"], t["height"])
    return ctf.Texture.latent_mlp(t["latent"], t["mlp"], t["width"], t["height"])


def run_gpu(ctf, tex, uv, grad, mode, fb, flags, E, filt, seed=0, frame_index=0):
    dt = dev_tex(ctf, tex)
    uvd = torch.from_numpy(np.ascontiguousarray(uv)).cuda()
    gd = None if grad is None else torch.from_numpy(np.ascontiguousarray(grad)).cuda()
    if uv.ndim == 4:
        out, rec = ctf.filter_batch(dt, uvd, gd, mode, fb, flags, seed, frame_index, filter=filt, max_evals=E)
    else:
        out, rec = ctf.filter_frame(dt, uvd, gd, mode, fb, flags, seed, frame_index, filter=filt, max_evals=E)
    torch.cuda.synchronize()
    return {"out": out.cpu().numpy(), "rec": rec.cpu().numpy().view(np.uint32)}


def run_oracle(tex, uv, grad, mode, fb, flags, E, filt, seed=0, frame_index=0):
    import oracle
    return oracle.filter_frame(tex, uv, grad, mode, fb, flags, seed, frame_index, debug=False, filter=filt,
                               max_evals=E)


def check(ctf, tex, uv, g, filt, seed, frame_index=0, modes=MODES):
    for mode, fb, fl, E in modes:
        o = run_oracle(tex, uv, g, mode, fb, fl, E, filt, seed, frame_index)
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, E, filt, seed, frame_index)
        what = f"filter={filt} mode={mode} fb={fb} flags={fl} E={E}"
        np.testing.assert_array_equal(gg["rec"], o["rec"], err_msg=f"records {what}")
        err = np.abs(gg["out"].astype(np.float64) - o["out"])
        assert err.max() <= ATOL, f"colour error {err.max()} {what}"


@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("mag,theta", [(4.0, 0.0), (3.0, 30.0), (2.0, 45.0)])
def test_uniform_quads(ctf, filt, mag, theta):
    """Magnified rotated quads: mostly exact waves (List / Box / Mask), E = 1 and 2."""
    tex = bc1_tex(64, 64, 3, "image")
    uv, g = synthetic.rotated_quad(64, 64, 64, 64, mag, theta, jitter_seed=1)
    check(ctf, tex, uv, g, filt, seed=5)


@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("mag,theta,cov", [(1.3, 33.0, "circle"), (0.7, 12.0, "halfplane"), (0.25, 70.0, None)])
def test_ragged_and_fallback_frames(ctf, filt, mag, theta, cov):
    """Partial waves (61x37 frame, coverage masks), clamp at the texture edge, fallback waves."""
    tex = bc1_tex(128, 128, 7, "image")
    uv, g = synthetic.rotated_quad(61, 37, 128, 128, mag, theta, coverage=cov, radius=16.0, jitter_seed=4)
    check(ctf, tex, uv, g, filt, seed=77, frame_index=3)


def test_random_uv_and_edges(ctf):
    """Random uv (every wave falls back; n saturates), out-of-range / infinite coordinates."""
    rng = np.random.default_rng(9)
    tex = bc1_tex(64, 32, 5, "random")
    uv = rng.random((21, 43, 2)).astype(np.float32)
    uv[rng.random((21, 43)) < 0.1, 0] = np.nan
    uv[0, :5] = [[-100.0, 3.0], [np.inf, 0.5], [0.5, -np.inf], [1.0, 1.0], [0.0, 0.0]]
    for filt in FILTERS:
        check(ctf, tex, uv, None, filt, seed=2**40 + 3)


def test_perspective_plane_batch(ctf):
    """Config-2-shaped perspective plane (small), two frames in one batched launch."""
    tex = bc1_tex(256, 256, 2, "image")
    uv = np.stack([synthetic.perspective_plane(96, 56, 256, 256, synthetic.PLANE_C2)[0],
                   synthetic.perspective_plane(96, 56, 256, 256, synthetic.PLANE_C4)[0]])
    for filt in FILTERS:
        for mode, fb, fl, E in [(3, 3, 0, 1), (3, 2, 0, 2), (0, 0, 0, 1)]:
            o = [run_oracle(tex, uv[f], None, mode, fb, fl, E, filt, 4, 10 + f) for f in range(2)]
            gg = run_gpu(ctf, tex, uv, None, mode, fb, fl, E, filt, 4, 10)
            for f in range(2):
                np.testing.assert_array_equal(gg["rec"][f], o[f]["rec"])
                assert np.abs(gg["out"][f].astype(np.float64) - o[f]["out"]).max() <= ATOL


def test_latent_mlp_bicubic(ctf):
    """The latent-MLP texture format through the bicubic kernel."""
    tex = mlp_tex(64, 64, 3)
    uv, g = synthetic.rotated_quad(40, 24, 64, 64, 2.5, 20.0, coverage="circle", radius=10.0)
    check(ctf, tex, uv, g, 2, seed=1,
          modes=[(0, 0, 0, 1), (1, 0, 0, 1), (3, 3, 0, 1), (3, 2, 0, 2), (4, 0, 0, 2), (3, 3, 2, 1)])


def test_exact_waves_equal_full_filter_bitwise(ctf):
    """An exact collaborative wave returns the full 16-tap filter bit for bit (same chain)."""
    tex = bc1_tex(128, 128, 1, "image")
    uv, g = synthetic.rotated_quad(64, 48, 128, 128, 2.6, 25.0)
    for filt in FILTERS:
        full = run_gpu(ctf, tex, uv, g, 0, 0, 0, 1, filt)
        col = run_gpu(ctf, tex, uv, g, 3, 3, 0, 2, filt)
        path = (col["rec"] >> 22) & 7
        px = np.repeat(np.repeat(path == 0, 4, 0), 8, 1)[:uv.shape[0], :uv.shape[1]]
        assert px.mean() > 0.5
        np.testing.assert_array_equal(col["out"][px], full["out"][px])


def test_unsupported_combinations(ctf):
    """WC with a bicubic filter and max_evals = 2 with bilinear are rejected (R-28)."""
    tex = dev_tex(ctf, bc1_tex(32, 32, 1, "image"))
    uv = torch.full((8, 8, 2), 0.5, device="cuda")
    for mode, fb, filt, E in [(2, 0, 1, 1), (3, 1, 2, 1), (3, 3, 0, 2)]:
        with pytest.raises(ctf.CtfError):
            ctf.filter_frame(tex, uv, None, mode, fb, filter=filt, max_evals=E)
