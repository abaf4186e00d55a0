"""Config-6 bicubic calls (4K perspective plane, BC1 4096^2) for ncu: Catmull-Rom List C+ E=2
then E=1, then the full 16-tap filter; and a timing line per variant.
usage: python scripts/prof_bicubic.py [lib.so ...]"""
import sys
import torch
sys.path.insert(0, ".")
import synthetic  # noqa: E402
import paper_2506_17770_b200.ctf as ctf  # noqa: E402

dev = torch.device("cuda")
T = 4096
tex = ctf.Texture.bc1(synthetic.bc1_texture(T, T, 0, "image"), T, T, device=dev)
uv, g = synthetic.perspective_plane_torch(3840, 2160, T, T, synthetic.PLANE_C2, device=dev)
out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device=dev)
rec = torch.empty((540, 480), dtype=torch.int32, device=dev)
libs = sys.argv[1:] or [None]
for lp in libs:
    if lp:
        ctf._lib = ctf.load_library(lp)
    for name, mode, fb, filt, E in (("cr_list_e2", 3, 3, 2, 2), ("cr_list_e1", 3, 3, 2, 1), ("cr_full16", 0, 0, 2, 1),
                                     ("bs_list_e2", 3, 3, 1, 2)):
        f = lambda: ctf.filter_frame(tex, uv, g, mode, fb, 0, 7, 0, out=out, rec=rec, filter=filt, max_evals=E)
        f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(lp or "in-tree", name, f"{ms:.3f} ms {3840 * 2160 / ms / 1e6:.2f} Gpix/s")
