"""Single-frame latency (configs 1 and 2): device time per ctf_filter_frame call, eager
(back-to-back Python calls) and CUDA-graph replay of G captured calls (no host overhead),
for the library's automatic launch choice and with CTF_FLAG_SEPARATE_PASSES."""
import sys

import torch

sys.path.insert(0, ".")
import synthetic  # noqa: E402
import paper_2506_17770_b200.ctf as ctf  # noqa: E402

libs = sys.argv[1:] or [None]
dev = torch.device("cuda")
cases = {}
b1 = synthetic.bc1_texture(32, 32, 7, "image")
u1, g1 = synthetic.rotated_quad(64, 64, 32, 32, 4.0, 30.0)
cases["c1_64x64"] = (b1, 32, torch.from_numpy(u1).to(dev), torch.from_numpy(g1).to(dev))
b2 = synthetic.bc1_texture(2048, 2048, 7, "image")
u2, g2 = synthetic.perspective_plane_torch(1920, 1080, 2048, 2048, synthetic.PLANE_C2, device=dev)
cases["c2_1080p"] = (b2, 2048, u2, g2)
for lp in libs:
    if lp:
        ctf._lib = ctf.load_library(lp)
    for name, (blocks, T, uv, g) in cases.items():
        tex = ctf.Texture.bc1(blocks, T, T, device=dev)
        hf, wf = uv.shape[:2]
        out = torch.empty((hf, wf, 4), dtype=torch.float32, device=dev)
        rec = torch.empty(((hf + 3) // 4, (wf + 7) // 8), dtype=torch.int32, device=dev)
        ws = ctf.workspace_for(tex, 3, 0, wf, hf, 1, dev)
        for sep in (0, ctf.FLAG_SEPARATE_PASSES):
            f = lambda: ctf.filter_frame(tex, uv, g, 3, 3, sep, 7, 0, out=out, rec=rec, workspace=ws)  # noqa: E731
            for _ in range(5):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 200
            e0.record()
            for _ in range(reps):
                f()
            e1.record()
            torch.cuda.synchronize()
            eager = e0.elapsed_time(e1) / reps * 1e3
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            G = 50
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                f()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr, stream=s):
                    for _ in range(G):
                        f()
            gr.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            graph = e0.elapsed_time(e1) / (10 * G) * 1e3
            print(f"{lp or 'in-tree'} {name} {'separate' if sep else 'auto    '}: eager {eager:7.2f} us/call  "
                  f"graph {graph:7.2f} us/call  ({wf * hf / graph / 1e3:.1f} Gpix/s in the graph)")
