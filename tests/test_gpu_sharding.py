"""SURVEY §8(e) sharding through the C ABI on one GPU (-m gpu): a frame split into wave-row
strips (ctf_params.row0) and a batch split into frame blocks give exactly the 1-call results —
records, producer ids, selections and colours bit for bit (waves never read another wave's
pixels; the RNG counter uses the frame row row0 + y)."""
import numpy as np
import pytest

import synthetic
from paper_2506_17770_b200 import dist as cdist
from tests.helpers import bc1_tex, mlp_tex

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2506_17770_b200.ctf as c
    c.load_library()
    return c


def _dev_tex(ctf, t):
    if t["format"] == 1:
        return ctf.Texture.bc1(t["bc1"], t["width"], t["height"])
    return ctf.Texture.latent_mlp(t["latent"], t["mlp"], t["width"], t["height"])


def _run(ctf, tex, uv, g, mode, fb, debug, row0=0, filt=0, frame_index=0, **kw):
    shape = uv.shape[:-1]
    dbg = None
    if debug:
        dbg = {"produced_id": torch.zeros(shape, dtype=torch.int32, device="cuda"),
               "selection": torch.zeros(shape, dtype=torch.int32, device="cuda"),
               "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
    out, rec = ctf.filter_batch(tex, uv, g, mode, fb, 0, 11, frame_index, debug=dbg, row0=row0, filter=filt, **kw)
    torch.cuda.synchronize()
    r = {"out": out.cpu(), "rec": rec.cpu()}
    if debug:
        r["pid"], r["sel"] = dbg["produced_id"].cpu(), dbg["selection"].cpu()
    return r


CASES = [("bc1_list_cplus", "bc1", 3, 3, 0, True), ("bc1_box_c", "bc1", 4, 2, 0, True),
         ("bc1_list_stf", "bc1", 3, 0, 0, True), ("bc1_bicubic_cr_cplus", "bc1", 3, 3, 2, False),
         ("mlp_list_cplus", "mlp", 3, 3, 0, True)]


@pytest.mark.parametrize("name,fmt,mode,fb,filt,debug", CASES)
@pytest.mark.parametrize("world", [2, 3, 5])
def test_strips_equal_whole_frame(ctf, name, fmt, mode, fb, filt, debug, world):
    W = 512
    t = bc1_tex(W, W, 4, "image") if fmt == "bc1" else mlp_tex(W, W, 4)
    tex = _dev_tex(ctf, t)
    F, Wf, Hf = 2, 200, 142             # ragged: 142 rows = 35.5 wave-rows, 25 wave-columns
    uv = torch.empty((F, Hf, Wf, 2), dtype=torch.float32)
    g = torch.empty((F, Hf, Wf, 4), dtype=torch.float16)
    for f in range(F):   # grazing plane: exact, fallback, partial and minified waves
        u, gg = synthetic.perspective_plane(Wf, Hf, W, W, synthetic.PLANE_C4, cam_height=1.0 + 0.3 * f)
        uv[f], g[f] = torch.from_numpy(u), torch.from_numpy(gg)
    uv, g = uv.cuda(), g.cuda()
    whole = _run(ctf, tex, uv, g, mode, fb, debug, filt=filt, frame_index=5)
    paths = ((whole["rec"].numpy().view(np.uint32) >> 22) & 7)
    assert (paths == 0).any() and ((paths >= 1) & (paths <= 4)).any()
    for r in range(world):
        row0, rows = cdist.strip_shard(Hf, world, r)
        part = _run(ctf, tex, uv[:, row0:row0 + rows].contiguous(), g[:, row0:row0 + rows].contiguous(), mode, fb,
                    debug, row0=row0, filt=filt, frame_index=5)
        wy0 = row0 // 4
        assert torch.equal(part["rec"], whole["rec"][:, wy0:wy0 + part["rec"].shape[1]]), (name, r)
        assert torch.equal(part["out"], whole["out"][:, row0:row0 + rows]), (name, r)
        if debug:
            assert torch.equal(part["pid"], whole["pid"][:, row0:row0 + rows])
            assert torch.equal(part["sel"], whole["sel"][:, row0:row0 + rows])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_frame_blocks_equal_whole_batch(ctf, world):
    W = 1024
    tex = _dev_tex(ctf, bc1_tex(W, W, 2, "image"))
    F, Wf, Hf = 8, 320, 180
    uv = torch.empty((F, Hf, Wf, 2), dtype=torch.float32)
    g = torch.empty((F, Hf, Wf, 4), dtype=torch.float16)
    for f in range(F):
        u, gg = synthetic.camera_path_frame(f, Wf, Hf, W, W, nframes=F)
        uv[f], g[f] = torch.from_numpy(u), torch.from_numpy(gg)
    uv, g = uv.cuda(), g.cuda()
    whole = _run(ctf, tex, uv, g, 3, 3, True, frame_index=0)
    for r in range(world):
        sh = cdist.frame_shard(F, world, r)
        part = _run(ctf, tex, uv[sh.start:sh.stop].contiguous(), g[sh.start:sh.stop].contiguous(), 3, 3, True,
                    frame_index=sh.start)
        for k in ("rec", "out", "pid", "sel"):
            assert torch.equal(part[k], whole[k][sh.start:sh.stop]), (k, r)


def test_row0_validation(ctf):
    tex = _dev_tex(ctf, bc1_tex(64, 64, 1, "image"))
    uv = torch.zeros((8, 8, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(ctf.CtfError):
        ctf.filter_frame(tex, uv, None, 3, 3, row0=2)     # not a multiple of 4
    with pytest.raises(ctf.CtfError):
        ctf.filter_frame(tex, uv, None, 3, 3, row0=-4)
