"""GPU (CUDA path through the C ABI) vs CPU oracle parity — run with -m gpu on a B200.

Bar (BASELINE.json north_star): bit-exact unique counts, producer lanes/ids,
evaluation counts, per-wave records and RNG-driven selections; |colour| error
<= 1e-5 absolute per fp32 channel.
"""
import numpy as np
import pytest

import synthetic
from tests.helpers import bc1_tex, mlp_tex

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ATOL = 1e-5


@pytest.fixture(scope="module")
def ctf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2506_17770_b200.ctf as c
    c.load_library()
    return c


def to_dev_tex(ctf, t):
    if t["format"] == 1:
        return ctf.Texture.bc1(t["bc1"], t["width"], t["height"])
    return ctf.Texture.latent_mlp(t["latent"], t["mlp"], t["width"], t["height"])


def run_gpu(ctf, tex, uv, grad, mode, fb=3, flags=0, seed=0, frame_index=0, batch=False):
    dt = to_dev_tex(ctf, tex)
    uvd = torch.from_numpy(np.ascontiguousarray(uv)).cuda()
    gd = None if grad is None else torch.from_numpy(np.ascontiguousarray(grad)).cuda()
    hf, wf = uv.shape[-3], uv.shape[-2]
    shape = uv.shape[:-1]
    dbg = {"produced_id": torch.zeros(shape, dtype=torch.int32, device="cuda"),
           "selection": torch.zeros(shape, dtype=torch.int32, device="cuda"),
           "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
    if batch or uv.ndim == 4:
        out, rec = ctf.filter_batch(dt, uvd, gd, mode, fb, flags, seed, frame_index, debug=dbg)
    else:
        out, rec = ctf.filter_frame(dt, uvd, gd, mode, fb, flags, seed, frame_index, debug=dbg)
    torch.cuda.synchronize()
    return {"out": out.cpu().numpy(), "rec": rec.cpu().numpy().view(np.uint32),
            "produced_id": dbg["produced_id"].cpu().numpy().view(np.uint32),
            "selection": dbg["selection"].cpu().numpy().view(np.uint32),
            "unread": int(dbg["unread"].item())}


def run_oracle(tex, uv, grad, mode, fb=3, flags=0, seed=0, frame_index=0):
    import oracle
    return oracle.filter_frame(tex, uv, grad, mode, fb, flags, seed, frame_index)


def assert_parity(g, o, what=""):
    np.testing.assert_array_equal(g["rec"], o["rec"], err_msg=f"records {what}")
    np.testing.assert_array_equal(g["produced_id"], o["produced_id"], err_msg=f"produced ids {what}")
    np.testing.assert_array_equal(g["selection"], o["selection"], err_msg=f"selections {what}")
    err = np.abs(g["out"].astype(np.float64) - o["out"])
    assert err.max() <= ATOL, f"colour error {err.max()} {what}"


MODES = [(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0), (3, 1, 0), (3, 2, 0), (3, 3, 0),
         (3, 0, 2), (3, 1, 2), (3, 2, 2), (3, 3, 2),
         (4, 3, 0), (4, 0, 0), (5, 2, 0), (5, 3, 0), (6, 3, 0), (6, 1, 0)]   # Box, Mask16, Mask11


@pytest.mark.parametrize("theta", [0.0, 30.0, 45.0])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config1_uniform_4x(ctf, theta, seed):
    """Config 1: 64x64 frame of a 32x32 BC1 texture at 4x magnification, every mode."""
    tex = bc1_tex(32, 32, seed, "image")
    uv, g = synthetic.rotated_quad(64, 64, 32, 32, 4.0, theta, jitter_seed=seed)
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, g, mode, fb, fl, seed=seed)
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=seed)
        assert_parity(gg, o, f"mode={mode} fb={fb} flags={fl}")
        assert gg["unread"] == 0


@pytest.mark.parametrize("mag,theta,cov", [(1.3, 33.0, "circle"), (1.05, 61.0, "halfplane"), (2.2, 45.0, None),
                                           (0.7, 12.0, "circle"), (0.3, 80.0, None)])
def test_ragged_mixed_frames(ctf, mag, theta, cov):
    """Partial waves (61x37 frame, coverage masks), exact + fallback waves, slow-path collect."""
    tex = bc1_tex(128, 128, 7, "image")
    uv, g = synthetic.rotated_quad(61, 37, 128, 128, mag, theta, coverage=cov, radius=16.0, jitter_seed=4)
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, g, mode, fb, fl, seed=77, frame_index=5)
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=77, frame_index=5)
        assert_parity(gg, o, f"m={mag} mode={mode} fb={fb} flags={fl}")
        assert gg["unread"] == 0


def test_random_uv_stress(ctf):
    """Uniform random uv: huge AABBs (sort path), random BC1 blocks (both modes)."""
    rng = np.random.default_rng(3)
    tex = bc1_tex(256, 128, 5, "random")
    uv = rng.random((45, 83, 2)).astype(np.float32)
    uv[rng.random((45, 83)) < 0.1, 0] = np.nan
    uv[0, :5] = [[-100.0, 3.0], [np.inf, 0.5], [0.5, -np.inf], [1.0, 1.0], [0.0, 0.0]]
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, None, mode, fb, fl, seed=2**40 + 17)
        gg = run_gpu(ctf, tex, uv, None, mode, fb, fl, seed=2**40 + 17)
        assert_parity(gg, o, f"mode={mode} fb={fb}")


def test_clustered_uv_edge_cases(ctf):
    """Waves whose lanes share footprints, single active lanes, clamp duplicates at borders."""
    W = H = 16
    tex = bc1_tex(W, H, 2, "image")
    uv = np.full((8, 24, 2), np.nan, np.float32)
    uv[0:4, 0:8] = (5.3 / W, 7.6 / H)                   # all lanes share one footprint
    for l in (1, 3, 5, 6, 7):
        uv[l // 8, 8 + l % 8] = (0.2, 0.9)               # edge-remap example lanes
    uv[2, 19] = (1.0, 7.6 / H)                           # single lane, clamped x: n=2 > a=1
    uv[4:8, 0:8] = (1.0, 1.0)                            # corner clamp: n = 1
    uv[5, 9] = (0.0, 0.0)
    uv[6, 17:20] = [(0.999, 0.001), (0.001, 0.999), (0.5, 0.5)]
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, None, mode, fb, fl, seed=1)
        gg = run_gpu(ctf, tex, uv, None, mode, fb, fl, seed=1)
        assert_parity(gg, o, f"mode={mode} fb={fb}")


@pytest.mark.parametrize("wf,hf", [(1, 1), (8, 4), (9, 5), (7, 3)])
def test_tiny_frames(ctf, wf, hf):
    tex = bc1_tex(32, 32, 1, "image")
    uv, g = synthetic.rotated_quad(wf, hf, 32, 32, 3.0, 20.0)
    for mode, fb, fl in MODES:
        assert_parity(run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=4), run_oracle(tex, uv, g, mode, fb, fl, seed=4))


def test_all_uncovered(ctf):
    tex = bc1_tex(32, 32, 1, "image")
    uv = np.full((12, 20, 2), np.nan, np.float32)
    for mode, fb, fl in MODES:
        assert_parity(run_gpu(ctf, tex, uv, None, mode, fb, fl), run_oracle(tex, uv, None, mode, fb, fl))


def test_perspective_mixed_minification(ctf):
    """Config-4 shape at small size: grazing plane with horizon, minified + magnified waves."""
    tex = bc1_tex(512, 512, 11, "image")
    uv, g = synthetic.perspective_plane(256, 144, 512, 512, synthetic.PLANE_C4)
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, g, mode, fb, fl, seed=3)
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=3)
        assert_parity(gg, o, f"mode={mode} fb={fb} flags={fl}")


@pytest.mark.parametrize("mode,fb,fl", [(0, 0, 0), (3, 3, 0), (3, 2, 2), (3, 3, 2), (1, 0, 0), (4, 3, 0), (5, 3, 0)])
def test_latent_mlp_texture(ctf, mode, fb, fl):
    """Config-3 format at small size: latent grid + MLP decode."""
    tex = mlp_tex(64, 64, 3)
    uv, g = synthetic.rotated_quad(45, 22, 64, 64, 2.5, 17.0, coverage="circle", radius=14.0)
    assert_parity(run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=6), run_oracle(tex, uv, g, mode, fb, fl, seed=6))


@pytest.mark.parametrize("mode", [3, 4, 5, 6])
def test_latent_mlp_release_lean_kernels(ctf, mode):
    """Latent MLP, release build (paired tensor-core decode) for List / Box / Mask: FULL waves
    (no coverage mask) at m ~ 1.3-1.6 rotated (exact and n > 32 / area > 32 waves) and a
    magnified interior, against the oracle."""
    import oracle
    tex = mlp_tex(64, 64, 3)
    dt = to_dev_tex(ctf, tex)
    for mag, theta in ((1.3, 30.0), (1.6, 45.0), (3.0, 10.0)):
        uv, g = synthetic.rotated_quad(64, 32, 64, 64, mag, theta)
        o = oracle.filter_frame(tex, uv, g, mode, 3, 0, 8, 2)
        out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, 3, 0, 8, 2)
        np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"], err_msg=f"m={mag}")
        assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL


def test_batch_equals_frames(ctf):
    """ctf_filter_batch over 3 frames == per-frame oracle with frame_index + f."""
    tex = bc1_tex(128, 128, 3, "image")
    frames = [synthetic.rotated_quad(40, 20, 128, 128, 1.2 + 0.5 * f, 10.0 * f) for f in range(3)]
    uv = np.stack([f[0] for f in frames])
    g = np.stack([f[1] for f in frames])
    gg = run_gpu(ctf, tex, uv, g, 3, 3, 0, seed=9, frame_index=100, batch=True)
    for f in range(3):
        o = run_oracle(tex, uv[f], g[f], 3, 3, 0, seed=9, frame_index=100 + f)
        assert_parity({k: (v[f] if isinstance(v, np.ndarray) else v) for k, v in gg.items()}, o, f"frame {f}")


def test_exact_waves_bitwise_equal_4tap(ctf):
    """T3: on every exact wave the collaborative result equals 4-tap bilinear bit for bit."""
    tex = bc1_tex(512, 512, 2, "image")
    uv, g = synthetic.perspective_plane(320, 180, 512, 512, synthetic.PLANE_C2)
    c = run_gpu(ctf, tex, uv, g, 3, 3)
    f = run_gpu(ctf, tex, uv, g, 0, 0)
    exact = ((c["rec"] >> 22) & 7) == 0
    px = np.repeat(np.repeat(exact, 4, 0), 8, 1)[:180, :320]
    assert px.mean() > 0.9
    assert np.array_equal(c["out"][px].view(np.uint32), f["out"][px].view(np.uint32))


def test_determinism(ctf):
    tex = bc1_tex(256, 256, 2, "image")
    uv, g = synthetic.perspective_plane(160, 90, 256, 256, synthetic.PLANE_C4)
    a = run_gpu(ctf, tex, uv, g, 3, 3, 0, seed=5)
    b = run_gpu(ctf, tex, uv, g, 3, 3, 0, seed=5)
    for k in ("out", "rec", "produced_id", "selection"):
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32))


def test_stats_match_oracle(ctf):
    import oracle
    tex = bc1_tex(512, 512, 2, "image")
    uv, g = synthetic.perspective_plane(256, 144, 512, 512, synthetic.PLANE_C4)
    dt = to_dev_tex(ctf, tex)
    uvd, gd = torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda()
    out, rec = ctf.filter_frame(dt, uvd, gd, 3, 3, seed=1)
    ref, _ = ctf.filter_frame(dt, uvd, gd, 0, 0)
    st = ctf.stats(rec, 256, 144, 1, out, ref)
    o = oracle.frame_stats(rec.cpu().numpy().view(np.uint32), out.cpu().numpy(), ref.cpu().numpy())
    for k in ("waves_live", "waves_partial", "waves_exact", "waves_fallback", "waves_magnified", "pixels_active",
              "pixels_in_magnified_waves", "texel_evals", "texel_evals_in_magnified_waves", "max_evals_per_lane",
              "max_unique_per_wave"):
        assert st[k] == o[k], k
    assert st["unique_hist"] == o["unique_hist"].tolist()
    assert st["err_pixels"] == 256 * 144
    np.testing.assert_allclose(st["sum_sq_err"], o["sum_sq_err"], rtol=1e-9)
    np.testing.assert_allclose(st["max_abs_err"], o["max_abs_err"], rtol=1e-6)
    # the records themselves match the oracle's
    orc = oracle.filter_frame(tex, uv, g, 3, 3, 0, seed=1)
    np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), orc["rec"])


def test_host_pipeline_matches_device(ctf):
    tex = bc1_tex(256, 256, 4, "image")
    fr = [synthetic.perspective_plane(96, 52, 256, 256, synthetic.PLANE_C4) for _ in range(5)]
    uv = torch.from_numpy(np.stack([f[0] for f in fr])).pin_memory()
    g = torch.from_numpy(np.stack([f[1] for f in fr])).pin_memory()
    dt = to_dev_tex(ctf, tex)
    out_h = torch.empty((5, 52, 96, 4), dtype=torch.float32).pin_memory()
    rec_h = torch.empty((5, 13, 12), dtype=torch.int32).pin_memory()
    pipe = ctf.HostPipeline(96, 52, 2, True)
    pipe.run(dt, uv, g, out_h, rec_h, 3, 3, seed=8, frame_index=3)
    out_d, rec_d = ctf.filter_batch(dt, uv.cuda(), g.cuda(), 3, 3, seed=8, frame_index=3)
    assert torch.equal(out_h, out_d.cpu()) and torch.equal(rec_h, rec_d.cpu())


def test_abi_errors(ctf):
    tex = bc1_tex(32, 32, 1, "image")
    dt = to_dev_tex(ctf, tex)
    uv = torch.zeros((4, 8, 2), device="cuda")
    with pytest.raises(ctf.CtfError) as e:
        ctf.filter_frame(dt, uv, None, 7)
    assert e.value.code == ctf.CTF_EINVAL
    big = torch.zeros(16, dtype=torch.float32, device="cuda")
    with pytest.raises(ctf.CtfError) as e:
        ctf.filter_frame(dt, big[1:].view(-1)[:8].view(4, 1, 2) if False else uv, None, 3,
                         out=torch.zeros(4 * 8 * 4 + 1, device="cuda")[1:].view(4, 8, 4))
    assert e.value.code == ctf.CTF_EALIGN
    bad = ctf.Texture(ctf.FMT_BC1, 30, 32, dt.data)
    with pytest.raises(ctf.CtfError) as e:
        ctf.filter_frame(bad, uv, None, 3)
    assert e.value.code == ctf.CTF_EINVAL


@pytest.mark.parametrize("mode,fb,fl", [(3, 3, 0), (3, 2, 0), (3, 0, 2), (0, 0, 0), (2, 0, 0), (4, 3, 0), (4, 1, 0),
                                        (5, 3, 0), (6, 2, 0)])
def test_release_kernel_matches_oracle(ctf, mode, fb, fl):
    """The non-debug kernel instantiation (what bench.py runs) against the oracle."""
    import oracle
    tex = bc1_tex(512, 512, 13, "image")
    uv, g = synthetic.perspective_plane(203, 117, 512, 512, synthetic.PLANE_C4)
    o = oracle.filter_frame(tex, uv, g, mode, fb, fl, seed=21, frame_index=2)
    dt = to_dev_tex(ctf, tex)
    out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb, fl, 21, 2)
    np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
    assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL


@pytest.mark.parametrize("fb,fl", [(3, 0), (2, 0), (1, 0), (0, 0), (3, 2)])
def test_workspace_lists_equal_record_scan(ctf, fb, fl):
    """BC1 COLLAB: the workspace work lists and the record-scan second passes give identical
    records, colours and debug outputs (mixed scene: exact, fallback, partial, minified waves)."""
    tex = bc1_tex(512, 512, 5, "image")
    uv, g = synthetic.perspective_plane(333, 141, 512, 512, synthetic.PLANE_C4)
    dt = to_dev_tex(ctf, tex)
    uvd, gd = torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda()
    res = []
    for ws in (True, None):
        dbg = {"produced_id": torch.zeros(uv.shape[:2], dtype=torch.int32, device="cuda"),
               "selection": torch.zeros(uv.shape[:2], dtype=torch.int32, device="cuda"),
               "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
        out, rec = ctf.filter_frame(dt, uvd, gd, 3, fb, fl, seed=11, debug=dbg, workspace=ws)
        out2, rec2 = ctf.filter_frame(dt, uvd, gd, 3, fb, fl, seed=11, workspace=ws)   # release kernels
        res.append([t.cpu().numpy().view(np.uint32) for t in (out, rec, dbg["produced_id"], dbg["selection"], out2, rec2)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)
    import oracle
    o = oracle.filter_frame(tex, uv, g, 3, fb, fl, seed=11)
    np.testing.assert_array_equal(res[0][1], o["rec"])


@pytest.mark.parametrize("center,mag,theta", [((0.0, 0.0), 1.1, 20.0), ((1.0, 0.5), 1.3, 45.0),
                                              ((0.5, 1.0), 0.45, 10.0), ((0.0, 1.0), 2.5, 70.0)])
def test_full_waves_at_texture_borders(ctf, center, mag, theta):
    """FULL waves (every lane covered) straddling the texture border: clamp-duplicate corners
    and merged weights in the lean exact / fallback kernels (n > 32 at m ~ 1, 128-bit windows
    at m < 1), all fallbacks, with and without the work-list workspace."""
    tex = bc1_tex(64, 64, 9, "image")
    uv, g = synthetic.rotated_quad(96, 48, 64, 64, mag, theta, center=center, jitter_seed=2)
    for mode, fb, fl in [(3, 0, 0), (3, 1, 0), (3, 2, 0), (3, 3, 0), (3, 3, 2), (3, 2, 2)]:
        o = run_oracle(tex, uv, g, mode, fb, fl, seed=5, frame_index=3)
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=5, frame_index=3)
        assert_parity(gg, o, f"c={center} m={mag} fb={fb} flags={fl}")
        dt = to_dev_tex(ctf, tex)
        out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb, fl, 5, 3,
                                    workspace=None)
        assert np.array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
        assert np.array_equal(out.cpu().numpy().view(np.uint32), gg["out"].view(np.uint32))


def test_exact_waves_with_128bit_windows(ctf):
    """FULL exact waves whose footprint AABB only fits a 16x8 or 32x4 window (n <= 32): they
    leave the lean exact kernel and take the fallback kernel's exact branch (4-word masks)."""
    W = H = 64
    tex = bc1_tex(W, H, 6, "image")
    uv = np.zeros((8, 24, 2), np.float32)
    lx = np.arange(8)
    for wx, (step, row) in enumerate([(2, 5.0), (4, 20.0), (3, 40.0)]):   # 16-wide, 32-wide, 24-wide
        for ly in range(4):
            uv[ly, wx * 8 + lx, 0] = (step * lx + 0.5) / W
            uv[ly, wx * 8 + lx, 1] = (row + 0.25) / H
            uv[4 + ly, wx * 8 + lx, 0] = (step * lx + 0.5 + ly % 2) / W       # two rows of footprints
            uv[4 + ly, wx * 8 + lx, 1] = (row + 0.25 + (ly // 2) * 3.0) / H
    import oracle
    for mode, fb, fl in [(3, 3, 0), (3, 0, 0), (3, 2, 2), (5, 3, 0), (6, 3, 0), (5, 1, 0), (4, 3, 0), (4, 2, 0)]:
        o = run_oracle(tex, uv, None, mode, fb, fl, seed=9)
        gg = run_gpu(ctf, tex, uv, None, mode, fb, fl, seed=9)
        assert_parity(gg, o, f"fb={fb} flags={fl}")
    o = oracle.filter_frame(tex, uv, None, 3, 3, 0, 9)
    n = (o["rec"] >> 8) & 255
    path = (o["rec"] >> 22) & 7
    assert (path[0] == 0).all() and (n[0] == 32).all()   # the first wave row is exact with n = 32


@pytest.mark.parametrize("wf,hf,mag,theta,cov", [(104, 40, 1.2, 30.0, "circle"), (104, 36, 0.9, 50.0, None),
                                                 (24, 8, 2.0, 10.0, None), (8, 12, 1.5, 60.0, "halfplane"),
                                                 (136, 44, 0.6, 15.0, "circle")])
def test_release_paired_runs(ctf, wf, hf, mag, theta, cov):
    """The release BC1 COLLAB kernel pairs consecutive waves of an interior run for one decode
    pass: odd-length runs (13, 3, 1, 17 waves), pairs mixing exact / fallback / partial /
    empty waves and nA + nB > 32 (two passes) give the oracle's records and colours, and the
    debug kernel's (unpaired) colours bit for bit."""
    import oracle
    tex = bc1_tex(128, 128, 17, "image")
    uv, g = synthetic.rotated_quad(wf, hf, 128, 128, mag, theta, coverage=cov, radius=14.0, jitter_seed=6)
    dt = to_dev_tex(ctf, tex)
    for mode, fb, fl in [(3, 3, 0), (3, 0, 0), (3, 2, 0)]:
        o = oracle.filter_frame(tex, uv, g, mode, fb, fl, seed=8, frame_index=1)
        out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb, fl, 8, 1)
        np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
        assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=8, frame_index=1)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), gg["out"].view(np.uint32))


@pytest.mark.parametrize("nf", [2, 3, 5])
def test_multi_frame_work_lists(ctf, nf):
    """A batched BC1 COLLAB call with a workspace (work lists over all frames of the batch):
    records, colours and debug outputs equal the record-scan path (no workspace) bit for bit
    and the per-frame oracle, for every fallback."""
    import oracle
    tex = bc1_tex(128, 128, 4, "image")
    frames = [synthetic.rotated_quad(64, 28, 128, 128, 0.8 + 0.35 * f, 17.0 * f, coverage="circle" if f % 2 else None,
                                     radius=12.0, jitter_seed=f) for f in range(nf)]
    uv = torch.from_numpy(np.stack([f[0] for f in frames])).cuda()
    g = torch.from_numpy(np.stack([f[1] for f in frames])).cuda()
    dt = to_dev_tex(ctf, tex)
    for fb, fl in [(3, 0), (0, 0), (2, 2)]:
        res = []
        for ws in (True, None):
            dbg = {"produced_id": torch.zeros(uv.shape[:3], dtype=torch.int32, device="cuda"),
                   "selection": torch.zeros(uv.shape[:3], dtype=torch.int32, device="cuda"),
                   "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
            out, rec = ctf.filter_batch(dt, uv, g, 3, fb, fl, 6, 40, debug=dbg, workspace=ws)
            out2, rec2 = ctf.filter_batch(dt, uv, g, 3, fb, fl, 6, 40, workspace=ws)   # release kernels
            torch.cuda.synchronize()
            res.append([t.cpu().numpy().view(np.uint32) for t in (out, rec, dbg["produced_id"], dbg["selection"],
                                                                   out2, rec2)])
        for a, b in zip(*res):
            assert np.array_equal(a, b)
        for f in range(nf):
            o = oracle.filter_frame(tex, frames[f][0], frames[f][1], 3, fb, fl, seed=6, frame_index=40 + f)
            np.testing.assert_array_equal(res[0][1][f], o["rec"])
            assert np.abs(res[0][0][f].view(np.float32).astype(np.float64) - o["out"]).max() <= ATOL


@pytest.mark.parametrize("wf,hf,mag,theta", [(104, 40, 1.5, 25.0), (136, 44, 0.9, 60.0)])
def test_release_paired_runs_latent_mlp(ctf, wf, hf, mag, theta):
    """The release latent-MLP COLLAB kernel decodes the texels of a CTA's waves as the rows of one
    tcgen05 tile (R-29, CTA-level collaboration): records equal the oracle's, colours are within
    the parity bar of the oracle and within 1e-6 of the debug kernel's (one wave per mma.sync
    decode: the same 3xFP16 products, another fp32 accumulation order), on odd runs with partial
    waves."""
    import oracle
    tex = mlp_tex(64, 64, 5)
    uv, g = synthetic.rotated_quad(wf, hf, 64, 64, mag, theta, coverage="circle", radius=15.0, jitter_seed=3)
    dt = to_dev_tex(ctf, tex)
    for mode, fb, fl in [(3, 3, 0), (3, 0, 0)]:
        o = oracle.filter_frame(tex, uv, g, mode, fb, fl, seed=12, frame_index=2)
        out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb, fl, 12, 2)
        np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
        assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL
        gg = run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=12, frame_index=2)
        np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), gg["rec"])
        assert np.abs(out.cpu().numpy().astype(np.float64) - gg["out"].astype(np.float64)).max() <= 1e-6


def anisotropic_quad(wf, hf, tex_w, tex_h, sx, sy, theta_deg, center=(0.5, 0.5)):
    """uv of a plane stretched by (sx, sy) texels per pixel and rotated by theta: thin slanted
    footprints whose AABB is wide while n stays <= 32 (a linear map, no RNG)."""
    yy, xx = np.mgrid[0:hf, 0:wf].astype(np.float64)
    px, py = xx + 0.5 - wf / 2, yy + 0.5 - hf / 2
    c, s = np.cos(np.radians(theta_deg)), np.sin(np.radians(theta_deg))
    tx, ty = c * sx * px - s * sy * py, s * sx * px + c * sy * py
    uv = np.stack([(tx + 0.37) / tex_w + center[0], (ty + 0.21) / tex_h + center[1]], -1).astype(np.float32)
    g = np.zeros((hf, wf, 4), np.float16)
    g[..., 0], g[..., 1], g[..., 2], g[..., 3] = c * sx, s * sx, -s * sy, c * sy
    return uv, g


@pytest.mark.parametrize("sx,sy,theta,center", [(1.4, 0.05, 10.0, (0.5, 0.5)), (1.5, 0.2, 15.0, (0.5, 0.5)),
                                                (1.3, 0.1, 5.0, (0.5, 0.5)), (2.6, 0.05, 0.0, (0.5, 0.0))])
def test_mask_and_box_variants_in_the_lean_kernels(ctf, sx, sy, theta, center):
    """Box and Mask 16x16 / 11x11 run the lean kernels (Box: AABB-order producers, AABB-area
    evaluations; both exact and fallback decided by its area test); Mask: FULL waves with n <= 32 whose AABB exceeds the
    grid (wide thin footprints; at the clamped top edge one texel row, so n <= 32 up to 32
    wide) must fall back in the lean fallback kernel exactly where the oracle's Mask test does,
    with and without the work-list workspace, debug and release builds."""
    import oracle
    W = H = 128
    tex = bc1_tex(W, H, 7, "image")
    uv, g = anisotropic_quad(64, 32, W, H, sx, sy, theta, center)
    lst = oracle.filter_frame(tex, uv, g, 3, 3, 0, 4)["rec"]
    rejected = 0
    for mode in (4, 5, 6):
        for fb in (3, 2, 0):
            o = run_oracle(tex, uv, g, mode, fb, 0, seed=4, frame_index=1)
            gg = run_gpu(ctf, tex, uv, g, mode, fb, 0, seed=4, frame_index=1)
            assert_parity(gg, o, f"mode={mode} fb={fb}")
            assert gg["unread"] == 0
            dt = to_dev_tex(ctf, tex)
            out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb, 0, 4, 1,
                                        workspace=None)
            np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
            assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL
        m = oracle.filter_frame(tex, uv, g, mode, 3, 0, 4)["rec"]
        if mode == 4:
            continue
        rejected += int(((((lst >> 22) & 7) == 0) & (((m >> 22) & 7) != 0)).sum())
    assert rejected > 0   # the scene exercises Mask's grid test on List-exact waves


def _tie_frames():
    """The measure-zero tie constructions of tests/test_oracle_pins.py (STF: u0 == s; C+ extra
    pick: u2 * wsum == w_0), several seeds each, as (uv, mode, fb, flags, seed)."""
    import oracle
    W = H = 16
    cases = []
    for seed in range(1, 400):
        r = oracle.philox4x32_10([0, 0, 0, 0], [seed, 0])
        u0, u1 = (int(r[0]) >> 8) / 2.0 ** 24, (int(r[1]) >> 8) / 2.0 ** 24
        if u1 < u0 < 0.5 and u1 + 2.0 ** -24 < 0.5:
            uv = np.full((4, 8, 2), np.nan, np.float32)
            uv[0, 0] = (np.float32((0.5 + u0) / W), np.float32((0.5 + u1 + 2.0 ** -24) / H))
            cases.append((uv, 1, 0, 0, seed))
            if len(cases) == 4:
                break
    nst = len(cases)
    for seed in range(1, 3000):
        u = [[(int(r[k]) >> 8) / 2.0 ** 24 for k in range(3)]
             for r in (oracle.philox4x32_10([x, 0, 0, 0], [seed, 0]) for x in range(3))]
        s_ = 1.0 - u[2][2]
        if 0.0 < s_ < 0.5 and all(ui[1] < 0.5 for ui in u) and {(1 if ui[0] < s_ else 0) + 2 for ui in u} == {2, 3}:
            uv = np.full((4, 8, 2), np.nan, np.float32)
            uv[0, 0:3] = (np.float32((0.5 + s_) / W), np.float32(1.0 / H))
            cases.append((uv, 3, 3, 2, seed))
            if len(cases) == nst + 4:
                break
    return cases


def test_rng_ties_match_oracle(ctf):
    """STF and C+ decisions at exact ties of the 2^-24 uniform grid (strict comparisons,
    P:460-461): debug kernels bitwise (records, producers, selections), release
    kernels records + colours."""
    tex = bc1_tex(16, 16, 2, "random")
    cases = _tie_frames()
    assert len(cases) == 8
    for uv, mode, fb, fl, seed in cases:
        o = run_oracle(tex, uv, None, mode, fb, fl, seed=seed)
        assert_parity(run_gpu(ctf, tex, uv, None, mode, fb, fl, seed=seed), o, f"tie m{mode} s{seed}")
        dt = to_dev_tex(ctf, tex)
        out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), None, mode, fb, fl, seed, 0)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
        assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL


@pytest.mark.parametrize("jac", [[[6.0, 0.0], [0.0, 1.0]], [[1.0, 0.5], [0.0, 12.0]], [[7.5, 0.0], [0.0, 15.0]],
                                 [[4.0, 3.0], [3.0, 4.0]], [[9.0, 0.0], [0.0, 3.0]], [[2.0, 0.0], [0.0, 23.0]]])
def test_big_window_waves(ctf, jac):
    """Minified waves whose footprint AABB exceeds the second kernel's 32 x 32 window: the third
    kernel's 64 x 64 window (AABBs up to 64 x 64) and, beyond it, the sort-based general path
    (9 x 3 and 2 x 23 texels per pixel: 65 texels wide / 71 tall).  Every mode and fallback,
    debug kernels bitwise, release kernels records + colours."""
    tex = bc1_tex(256, 256, 5, "image")
    uv, g = synthetic.affine_quad(48, 20, 256, 256, jac)
    for mode, fb, fl in MODES:
        o = run_oracle(tex, uv, g, mode, fb, fl, seed=9)
        assert_parity(run_gpu(ctf, tex, uv, g, mode, fb, fl, seed=9), o, f"jac={jac} mode={mode} fb={fb} fl={fl}")
        if mode == 3:
            assert_parity(run_gpu(ctf, tex, uv, g, mode, fb, fl | ctf.FLAG_SEPARATE_PASSES, seed=9), o,
                          f"separate jac={jac} fb={fb} fl={fl}")
        # the single fused launch (small call) and the separate passes (lean kernel, then the
        # third and the wide-window kernels side by side, AABB-routed work lists)
        for sep in (0, ctf.FLAG_SEPARATE_PASSES):
            dt = to_dev_tex(ctf, tex)
            out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), mode, fb,
                                        fl | sep, 9, 0)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(rec.cpu().numpy().view(np.uint32), o["rec"])
            assert np.abs(out.cpu().numpy().astype(np.float64) - o["out"]).max() <= ATOL
