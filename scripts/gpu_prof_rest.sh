# ncu source-level capture of the lean fallback kernel (config-4 scene, C+ call) — run under gpurun
set -x
mkdir -p gpurun_out
TAG=${TAG:-fb}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_rest_kernel -s 10 -c 1 \
    -o gpurun_out/prof_fb_$TAG python scripts/prof_c4.py > gpurun_out/ncu_fb_$TAG.log 2>&1
tail -3 gpurun_out/ncu_fb_$TAG.log
ncu -i gpurun_out/prof_fb_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_fb_${TAG}_details.csv 2>/dev/null
python - <<PY
import torch, sys
sys.path.insert(0, ".")
import synthetic, numpy as np
import paper_2506_17770_b200.ctf as ctf
T, Wf, Hf = 4096, 3840, 2160
tex = ctf.Texture.bc1(synthetic.bc1_texture(T, T, 0, "image"), T, T, device="cuda")
uv, g = synthetic.perspective_plane_torch(Wf, Hf, T, T, synthetic.PLANE_C4, device="cuda")
out, rec = ctf.filter_frame(tex, uv, g, 3, 3, 0, 1, 0)
r = rec.cpu().numpy().view(np.uint32).reshape(-1)
path = (r >> 22) & 7; a = (r >> 16) & 63
print("waves", r.size, "C+ full", int(((path == 4) & (a == 32)).sum()), "C+ partial", int(((path == 4) & (a < 32) & (a > 0)).sum()))
PY
