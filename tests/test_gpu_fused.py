"""The single-launch fused kernel (BC1 collaborative bilinear calls of <= 131072 waves) and the
multi-kernel pipeline (CTF_FLAG_SEPARATE_PASSES) give identical results — records, producer
ids, STF / C+ selections and colours bit for bit — and both match the oracle (-m gpu)."""
import numpy as np
import pytest

import synthetic
from tests.helpers import bc1_tex

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2506_17770_b200.ctf as c
    c.load_library()
    return c


def _run(ctf, tex, uv, g, mode, fb, flags):
    shape = uv.shape[:-1]
    dbg = {"produced_id": torch.zeros(shape, dtype=torch.int32, device="cuda"),
           "selection": torch.zeros(shape, dtype=torch.int32, device="cuda"),
           "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
    out, rec = ctf.filter_frame(tex, uv, g, mode, fb, flags, 5, 2, debug=dbg)
    torch.cuda.synchronize()
    assert int(dbg["unread"].item()) == 0
    return {"out": out.cpu().numpy(), "rec": rec.cpu().numpy().view(np.uint32),
            "produced_id": dbg["produced_id"].cpu().numpy().view(np.uint32),
            "selection": dbg["selection"].cpu().numpy().view(np.uint32)}


SCENES = {
    "grazing": lambda W: synthetic.perspective_plane(333, 150, W, W, synthetic.PLANE_C4),
    "camera0": lambda W: synthetic.camera_path_frame(0, 320, 180, W, W),
    "minified_quad": lambda W: synthetic.rotated_quad(96, 40, W, W, 0.45, 17.0, coverage="circle", radius=30.0),
}


@pytest.mark.parametrize("scene", sorted(SCENES))
@pytest.mark.parametrize("mode,fb,force", [(3, 3, 0), (3, 0, 0), (3, 1, 0), (3, 2, 0), (4, 3, 0), (5, 3, 0),
                                           (6, 2, 0), (3, 3, 1)])
def test_fused_equals_separate_and_oracle(ctf, scene, mode, fb, force):
    import oracle
    W = 1024
    t = bc1_tex(W, W, 6, "image")
    tex = ctf.Texture.bc1(t["bc1"], W, W)
    uv, g = SCENES[scene](W)
    uvd, gd = torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda()
    flags = ctf.FLAG_FORCE_FALLBACK if force else 0
    fused = _run(ctf, tex, uvd, gd, mode, fb, flags)
    sep = _run(ctf, tex, uvd, gd, mode, fb, flags | ctf.FLAG_SEPARATE_PASSES)
    for k in ("rec", "out", "produced_id", "selection"):
        np.testing.assert_array_equal(fused[k], sep[k], err_msg=k)
    o = oracle.filter_frame(t, uv, g, mode, fb, flags, 5, 2)
    for k in ("rec", "produced_id", "selection"):
        np.testing.assert_array_equal(fused[k], o[k], err_msg=k)
    assert float(np.abs(fused["out"].astype(np.float64) - o["out"]).max()) <= 1e-5
    paths = (fused["rec"] >> 22) & 7
    if not force:
        assert (paths == 0).any()


def test_fused_release_build_matches_separate(ctf):
    """Release kernels (no debug outputs): the fused single launch and the separate passes agree
    on records and colours for a frame with exact, fallback, partial and wide waves."""
    W = 2048
    t = bc1_tex(W, W, 3, "image")
    tex = ctf.Texture.bc1(t["bc1"], W, W)
    uv, g = synthetic.perspective_plane(640, 360, W, W, synthetic.PLANE_C4)
    uvd, gd = torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda()
    a = ctf.filter_frame(tex, uvd, gd, 3, 3, 0, 9, 0)
    b = ctf.filter_frame(tex, uvd, gd, 3, 3, ctf.FLAG_SEPARATE_PASSES, 9, 0)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
