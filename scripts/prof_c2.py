import sys, torch
sys.path.insert(0, ".")
import synthetic
import paper_2506_17770_b200.ctf as ctf
dev = torch.device("cuda")
b2 = synthetic.bc1_texture(2048, 2048, 7, "image")
tex = ctf.Texture.bc1(b2, 2048, 2048, device=dev)
u2, g2 = synthetic.perspective_plane_torch(1920, 1080, 2048, 2048, synthetic.PLANE_C2, device=dev)
out = torch.empty((1080, 1920, 4), dtype=torch.float32, device=dev)
rec = torch.empty((270, 240), dtype=torch.int32, device=dev)
for _ in range(5):
    ctf.filter_frame(tex, u2, g2, 3, 3, 0, 7, 0, out=out, rec=rec)
torch.cuda.synchronize()
