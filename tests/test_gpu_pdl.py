"""Programmatic dependent launch (PDL) ordering (-m gpu).

The lean kernels are launched as programmatic dependents of whatever precedes them on the
stream and wait for it in-kernel (griddepcontrol.wait) before their first global access;
small grids let the next kernel launch at once; the BC1 pipeline runs the third kernel and the
wide-window kernel side by side.  These tests check that results never depend on that
overlap: inputs written by a preceding kernel right before each call are the ones filtered,
an output buffer read by the next kernel holds the finished result, and back-to-back calls
captured in a CUDA graph equal the same calls made eagerly, bit for bit.
"""
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


def _frames(n, wf, hf, W):
    """n different frames of the camera path (torch, on the device)."""
    uvs, gs = [], []
    for f in range(n):
        u, g = synthetic.camera_path_frame_torch(8 * f, wf, hf, W, W)
        uvs.append(u)
        gs.append(g)
    torch.cuda.synchronize()   # the inputs are complete before any other stream reads them
    return uvs, gs


@pytest.mark.parametrize("wf,hf,flags", [(64, 64, 0), (320, 180, 0), (1920, 1080, 0), (3840, 2160, 0),
                                         (320, 180, 4)])
def test_inputs_written_just_before_the_call(ctf, wf, hf, flags):
    """Each call's input buffer is overwritten by a torch kernel immediately before the call
    (same stream); the call must filter the new contents.  The output of call k is consumed
    (copied) by a torch kernel right after it, before call k + 1 writes the same buffer."""
    W = 1024
    tex = ctf.Texture.bc1(bc1_tex(W, W, 3, "image")["bc1"], W, W)
    uvs, gs = _frames(4, wf, hf, W)
    uv = torch.empty_like(uvs[0])
    g = torch.empty_like(gs[0])
    out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device="cuda")
    rec = torch.empty(((hf + 3) // 4, (wf + 7) // 8), dtype=torch.int32, device="cuda")
    got = []
    for k in range(4):
        uv.copy_(uvs[k])
        g.copy_(gs[k])
        ctf.filter_frame(tex, uv, g, 3, 3, flags, 11, k, out=out, rec=rec)
        got.append((out.clone(), rec.clone()))   # read by the next kernel on the stream
    torch.cuda.synchronize()
    for k in range(4):
        o, r = ctf.filter_frame(tex, uvs[k].clone(), gs[k].clone(), 3, 3, flags, 11, k)
        torch.cuda.synchronize()
        assert torch.equal(got[k][1], r), k
        assert torch.equal(got[k][0], o), k


@pytest.mark.parametrize("wf,hf", [(64, 64), (1920, 1080)])
def test_graph_of_back_to_back_calls_equals_eager(ctf, wf, hf):
    """Single-frame calls captured in a CUDA graph (PDL edges between them) equal eager calls."""
    W = 1024
    tex = ctf.Texture.bc1(bc1_tex(W, W, 4, "image")["bc1"], W, W)
    uvs, gs = _frames(6, wf, hf, W)
    outs = [torch.empty(uvs[0].shape[:-1] + (4,), dtype=torch.float32, device="cuda") for _ in range(6)]
    recs = [torch.empty(((hf + 3) // 4, (wf + 7) // 8), dtype=torch.int32, device="cuda") for _ in range(6)]
    ws = ctf.workspace_for(tex, 3, 0, wf, hf, 1, "cuda")
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    call = lambda k: ctf.filter_frame(tex, uvs[k], gs[k], 3, 3, 0, 5, k, out=outs[k], rec=recs[k],
                                      stream=stream, workspace=ws)
    with torch.cuda.stream(stream):
        for k in range(6):   # warm-up (eager) and the reference results
            call(k)
    torch.cuda.synchronize()
    ref = [(o.clone(), r.clone()) for o, r in zip(outs, recs)]
    for o in outs:
        o.fill_(-1.0)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for k in range(6):
            call(k)
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    for k in range(6):
        assert torch.equal(recs[k], ref[k][1]), k
        assert torch.equal(outs[k], ref[k][0]), k
