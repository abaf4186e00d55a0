import sys, numpy as np, torch
sys.path.insert(0, '.')
import synthetic, oracle
from tests.helpers import bc1_tex
import paper_2506_17770_b200.ctf as ctf
if len(sys.argv) > 1:
    ctf._lib = ctf.load_library(sys.argv[1])
from oracle.oracle import decode_record
tex = bc1_tex(128, 128, 7, "image")
uv, g = synthetic.rotated_quad(61, 37, 128, 128, 0.3, 80.0, coverage=None, radius=16.0, jitter_seed=4)
o = oracle.filter_frame(tex, uv, g, 3, 0, 0, seed=77, frame_index=5)
dt = ctf.Texture.bc1(tex["bc1"], 128, 128)
dbg = {"produced_id": torch.zeros(uv.shape[:2], dtype=torch.int32, device="cuda"),
       "selection": torch.zeros(uv.shape[:2], dtype=torch.int32, device="cuda"),
       "unread": torch.zeros(1, dtype=torch.int32, device="cuda")}
for rep in range(3):
    out, rec = ctf.filter_frame(dt, torch.from_numpy(uv).cuda(), torch.from_numpy(g).cuda(), 3, 0, 0, 77, 5, debug=dbg if rep else None)
    r = rec.cpu().numpy().view(np.uint32)
    print('rep', rep, 'mismatches', int((r != o['rec']).sum()))
r = rec.cpu().numpy().view(np.uint32)
bad = np.argwhere(r != o["rec"])
for wy, wx in bad:
    print(wy, wx, {k: int(v[wy, wx]) for k, v in decode_record(r).items()}, {k: int(v[wy, wx]) for k, v in decode_record(o["rec"]).items()})
