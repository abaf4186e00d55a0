"""A/B timing of libctf builds on the bench workload (config 5 camera path, BC1 4K frames).

python scripts/time_libs.py [--frames F] [--mode M] [--fb B] lib_a.so lib_b.so ...
Libraries are timed interleaved (a, b, ..., a, b, ...) so clock drift hits all alike.
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import synthetic  # noqa: E402
import paper_2506_17770_b200.ctf as ctf  # noqa: E402
from paper_2506_17770_b200 import dist as cdist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=64)
ap.add_argument("--mode", type=int, default=3)
ap.add_argument("--fb", type=int, default=3)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--scene", default="c5", choices=["c5", "c4", "c2"])
ap.add_argument("--separate", action="store_true", help="CTF_FLAG_SEPARATE_PASSES")
ap.add_argument("libs", nargs="+")
a = ap.parse_args()

dev = torch.device("cuda")
libs = [ctf.load_library(p) for p in a.libs]
ctf._lib = libs[0]
F, Wf, Hf, T = a.frames, 3840, 2160, 4096
if a.scene == "c2":
    Wf, Hf = 1920, 1080
tex = ctf.Texture.bc1(synthetic.bc1_texture(T, T, 0, "image"), T, T, device=dev)
frames, base = cdist.weak_frames(F, 0)
uv = torch.empty((F, Hf, Wf, 2), dtype=torch.float32, device=dev)
grad = torch.empty((F, Hf, Wf, 4), dtype=torch.float16, device=dev)
for i, f in enumerate(frames):
    if a.scene == "c5":
        u, g = synthetic.camera_path_frame_torch(f, Wf, Hf, T, T, device=dev)
    elif a.scene == "c4":  # config-4 grazing plane, the same frame F times
        u, g = synthetic.perspective_plane_torch(Wf, Hf, T, T, synthetic.PLANE_C4, device=dev)
    else:  # config-2 shape: 1080p perspective plane
        u, g = synthetic.perspective_plane_torch(Wf, Hf, T, T, synthetic.PLANE_C2, device=dev)
    uv[i].copy_(u)
    grad[i].copy_(g)
out = torch.empty((F, Hf, Wf, 4), dtype=torch.float32, device=dev)
rec = torch.empty((F, (Hf + 3) // 4, (Wf + 7) // 8), dtype=torch.int32, device=dev)
res = {p: [] for p in a.libs}
outs = {}
for r in range(a.rounds):
    for p, lib in zip(a.libs, libs):
        ctf._lib = lib
        f = lambda: ctf.filter_batch(tex, uv, grad, a.mode, a.fb, 4 if a.separate else 0, 0, base, out=out, rec=rec)
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[p].append(e0.elapsed_time(e1) / a.reps)
        if r == 0:
            outs[p] = (out.clone(), rec.clone())
ref = outs[a.libs[0]]
for p in a.libs:
    ms = min(res[p])
    same = torch.equal(outs[p][0], ref[0]) and torch.equal(outs[p][1], ref[1])
    print(f"{p}: min {ms:.3f} ms  {F * Wf * Hf / ms / 1e6:.2f} Gpix/s  all {['%.3f' % x for x in res[p]]}  "
          f"identical_to_first={same}")
