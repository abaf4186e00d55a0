"""CPU checks of the boundary: libctf.so loads, exports every symbol include/ctf.h
declares, the product path never touches the oracle, and there is no CPU fallback."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "ctf.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ctf_[a-z_0-9]+)\s*\(", text)) - {"ctf_status"})


def test_library_exports_every_declared_symbol():
    from paper_2506_17770_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(str(lib_path))
    names = header_functions()
    assert {"ctf_filter_frame", "ctf_stats", "ctf_filter_batch"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    lib.ctf_abi_version.restype = ctypes.c_int
    assert lib.ctf_abi_version() == 6


def test_binding_declares_all_exports():
    import paper_2506_17770_b200.ctf as c
    assert sorted(c.EXPORTS) == header_functions()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2506_17770_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h")):
        src = p.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), p
        assert "ctf_oracle" not in src, p


def test_oracle_never_includes_product():
    src = (ROOT / "oracle" / "ctf_oracle.c").read_text()
    assert "#include \"" not in src and "ctf.h" not in src
    py = (ROOT / "oracle" / "oracle.py").read_text()
    assert "paper_2506_17770_b200" not in py


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    import paper_2506_17770_b200.ctf as c
    with pytest.raises((ValueError, RuntimeError)):
        c._ptr(torch.zeros(4))


def test_validation_errors_without_gpu():
    """Host-side validation runs before any CUDA call, so it is testable on CPU."""
    import paper_2506_17770_b200.ctf as c
    lib = c.load_library()
    tex = c.ctf_texture(1, 32, 32, 0, 0x1000, None, None)
    p = c.ctf_params(3, 3, 0, 0, 0)
    V = ctypes.c_void_p
    # null uv
    assert lib.ctf_filter_frame(ctypes.byref(tex), None, None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EINVAL
    # misaligned out
    assert lib.ctf_filter_frame(ctypes.byref(tex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1008), V(0x1000), None, None) == c.CTF_EALIGN
    # bad mode / dims / unsupported size
    p.mode = 9
    assert lib.ctf_filter_frame(ctypes.byref(tex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EINVAL
    p.mode = 3
    tex.width = 30
    assert lib.ctf_filter_frame(ctypes.byref(tex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EINVAL
    tex.width, tex.height = 8192, 8192
    assert lib.ctf_filter_frame(ctypes.byref(tex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EUNSUPPORTED
    tex.width, tex.height = 32, 32
    # ABI 6: strip origin row0 must be a non-negative multiple of 4; reserved_ must be 0
    for row0, res in ((2, 0), (-4, 0), (0, 1)):
        p.row0, p.reserved_ = row0, res
        assert lib.ctf_filter_frame(ctypes.byref(tex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EINVAL
    p.row0, p.reserved_ = 0, 0
    # ABI 6: the latent-MLP format requires the host copy of the weights (no hidden device
    # round trip / synchronisation in the launch path)
    mtex = c.ctf_texture(2, 32, 32, 0, 0x1000, 0x1000, None)
    assert lib.ctf_filter_frame(ctypes.byref(mtex), V(0x1000), None, 8, 4, ctypes.byref(p), V(0x1000), V(0x1000), None, None) == c.CTF_EINVAL
    lib.ctf_launches_per_call.argtypes = [ctypes.c_int32] * 6 + [ctypes.c_int]
    L = lib.ctf_launches_per_call
    # BC1 COLLAB bilinear, 4K frames (259200 waves per frame > 131072): exact, wide-window and
    # general kernels per pass; small passes (<= 131072 waves): one fused kernel
    assert L(1, 3, 0, 3840, 2160, 64, 1) == 3 and L(1, 3, 0, 3840, 2160, 64, 0) == 192
    assert L(1, 3, 0, 1920, 1080, 1, 0) == 1 and L(1, 3, 0, 1920, 1080, 4, 0) == 4      # 64800 waves: fused
    assert L(1, 3, 0, 1920, 1080, 4, 1) == 3                                              # batched: 259200 waves
    assert L(1, 3, 0, 1920, 1080, 1, 4) == 3                                              # separate passes asked
    assert L(1, 0, 0, 3840, 2160, 64, 1) == 1 and L(2, 3, 0, 64, 64, 8, 0) == 16
    assert L(2, 4, 0, 64, 64, 8, 1) == 2   # Box: lean exact + general (latent MLP)
    assert L(3, 3, 0, 64, 64, 1, 1) == -1 and L(1, 3, 0, 0, 64, 1, 1) == -1
    # the workspace flag does not change the count
    assert L(1, 3, 0, 3840, 2160, 64, 3) == 3 and L(2, 3, 0, 3840, 2160, 64, 3) == 2
    assert L(1, 3, 1, 3840, 2160, 64, 3) == 1   # bicubic: one kernel


def test_workspace_and_launch_accounting_per_mode():
    """Host logic: which modes take the lean kernels' work-list workspace and how many launches
    a call makes (List / Box / Mask: lean exact + lean fallback + general for BC1, lean exact +
    general for the latent MLP; every other mode: one general kernel)."""
    import torch
    import paper_2506_17770_b200.ctf as ctf
    bc1 = ctf.Texture.bc1(torch.zeros(8 * 64, dtype=torch.uint8), 32, 32, device="cpu")
    mlp = ctf.Texture(ctf.FMT_LATENT_MLP, 32, 32, torch.zeros(8 * 8 * 8, dtype=torch.float16))
    for mode in range(7):
        lean_bc1 = mode in (ctf.MODE_COLLAB, ctf.MODE_BOX, ctf.MODE_MASK16, ctf.MODE_MASK11)
        lean_mlp = lean_bc1
        assert (ctf.workspace_for(bc1, mode, 0, 64, 32, 2, "cpu") is not None) == lean_bc1, mode
        assert (ctf.workspace_for(mlp, mode, 0, 64, 32, 2, "cpu") is not None) == lean_mlp, mode
        assert ctf.launches_per_call(ctf.FMT_BC1, mode, 0, 1) == (3 if lean_bc1 else 1), mode
        assert ctf.launches_per_call(ctf.FMT_BC1, mode, 0, 1, wf=64, hf=64) == 1, mode   # fused when lean
        assert ctf.launches_per_call(ctf.FMT_LATENT_MLP, mode, 0, 1) == (2 if lean_mlp else 1), mode
        assert ctf.workspace_for(bc1, mode, 1, 64, 32, 2, "cpu") is None   # bicubic: no work lists


def test_binding_rejects_mismatched_buffers():
    """ctf.check_buffers (called by filter_frame / filter_batch / HostPipeline.run before the C
    call): an undersized, mistyped or foreign-device buffer raises instead of reaching the
    kernels, which take plain pointers and would read or write past its end."""
    torch = pytest.importorskip("torch")
    import paper_2506_17770_b200.ctf as c
    F, H, W = 2, 9, 13   # ragged: 3 wave-rows x 2 wave-columns per frame
    uv = torch.zeros((F, H, W, 2), dtype=torch.float32)
    g = torch.zeros((F, H, W, 4), dtype=torch.float16)
    out = torch.zeros((F, H, W, 4), dtype=torch.float32)
    rec = torch.zeros((F, 3, 2), dtype=torch.int32)
    c.check_buffers(uv, g, out, rec)                                          # exact sizes
    c.check_buffers(uv, None, out.flatten(), torch.zeros(100, dtype=torch.int32))   # flat, larger
    c.check_buffers(uv, g, out, None)                                        # host pipeline: no records
    dbg = {"produced_id": torch.zeros(F * H * W, dtype=torch.int32),
           "selection": torch.zeros(F * H * W, dtype=torch.int32), "unread": torch.zeros(1, dtype=torch.int32)}
    c.check_buffers(uv, g, out, rec, dbg)
    bad = [
        (uv.double(), g, out, rec, None),                       # uv dtype
        (uv[..., :1].contiguous(), g, out, rec, None),          # uv last dim
        (uv[0], g, out, rec, None),                             # uv rank
        (uv, g.float(), out, rec, None),                        # grad dtype
        (uv, g[:1], out, rec, None),                            # grad frames
        (uv, g, out[:, :-1], rec, None),                        # out too small
        (uv, g, out.half(), rec, None),                         # out dtype
        (uv, g, out, rec[:, :-1], None),                        # rec too small
        (uv, g, out, rec.float(), None),                        # rec dtype
        (uv, g, out.transpose(1, 2), rec, None),                # out not contiguous
        (uv, g, out, rec, dict(dbg, produced_id=torch.zeros(F * H * W - 1, dtype=torch.int32))),
        (uv, g, out, rec, dict(dbg, unread=torch.zeros(0, dtype=torch.int32))),
        (uv, g, out, torch.zeros((F, 3, 2), dtype=torch.int32, device="meta"), None),   # other device
    ]
    for args in bad:
        with pytest.raises(ValueError):
            c.check_buffers(*args)
