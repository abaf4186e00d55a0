"""Config-6 latent-MLP bicubic calls (4K perspective plane, latent 4096^2 texture):
Catmull-Rom List C+ E=2 / E=1 timings per library.  usage: python scripts/prof_bicubic_mlp.py [lib.so ...]"""
import sys
import torch
sys.path.insert(0, ".")
import synthetic  # noqa: E402
import paper_2506_17770_b200.ctf as ctf  # noqa: E402

dev = torch.device("cuda")
T = 4096
tex = ctf.Texture.latent_mlp(synthetic.latent_texture(T, T, 7), synthetic.mlp_weights(8), T, T, device=dev)
uv, g = synthetic.perspective_plane_torch(3840, 2160, T, T, synthetic.PLANE_C2, device=dev)
out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device=dev)
rec = torch.empty((540, 480), dtype=torch.int32, device=dev)
for lp in sys.argv[1:] or [None]:
    if lp:
        ctf._lib = ctf.load_library(lp)
    for name, mode, fb, filt, E in (("cr_list_e2", 3, 3, 2, 2), ("cr_list_e1", 3, 3, 2, 1)):
        f = lambda: ctf.filter_frame(tex, uv, g, mode, fb, 0, 7, 0, out=out, rec=rec, filter=filt, max_evals=E)
        f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5):
            f()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(lp or "in-tree", name, f"{ms:.3f} ms {3840 * 2160 / ms / 1e6:.2f} Gpix/s")
