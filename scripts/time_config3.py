"""Time config 3 (4K latent-MLP COLLAB) for a given libctf build: python scripts/time_config3.py [lib.so]"""
import sys, torch
sys.path.insert(0, '.')
import synthetic
import paper_2506_17770_b200.ctf as ctf
if len(sys.argv) > 1:
    ctf._lib = ctf.load_library(sys.argv[1])
dev = torch.device("cuda")
t3 = ctf.Texture.latent_mlp(synthetic.latent_texture(4096, 4096, 7), synthetic.mlp_weights(8), 4096, 4096, device=dev)
uv, g = synthetic.perspective_plane_torch(3840, 2160, 4096, 4096, synthetic.PLANE_C2, device=dev)
for mode in (3, 0):
    out = torch.empty(uv.shape[:-1] + (4,), device=dev); rec = torch.empty((540, 480), dtype=torch.int32, device=dev)
    f = lambda: ctf.filter_frame(t3, uv, g, mode, 3, 0, 7, 0, out=out, rec=rec)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); [f() for _ in range(10)]; b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(sys.argv[1:] or ["default"], "mode", mode, f"{ms:.3f} ms", f"{3840*2160/ms/1e6:.2f} Gpix/s")
