"""One config-4 (grazing plane, 4K, BC1 4096^2) COLLAB call per fallback, for ncu launch lists."""
import sys
import torch
sys.path.insert(0, ".")
import synthetic  # noqa: E402
import paper_2506_17770_b200.ctf as ctf  # noqa: E402

dev = torch.device("cuda")
T, Wf, Hf = 4096, 3840, 2160
tex = ctf.Texture.bc1(synthetic.bc1_texture(T, T, 0, "image"), T, T, device=dev)
uv, g = synthetic.perspective_plane_torch(Wf, Hf, T, T, synthetic.PLANE_C4, device=dev)
for fb in (0, 3):
    for _ in range(3):
        ctf.filter_frame(tex, uv, g, 3, fb, 0, 1, 0)
torch.cuda.synchronize()
