#!/usr/bin/env python
"""bench.py — throughput of the collaborative texture filtering hot path on B200.

Headline workload (BASELINE.json configs[4], "config 5"): a batch of 64 4K
(3840x2160) frames of the animated camera path over the perspective ground
plane (synthetic.camera_path_frame: magnification ~0.5-9.4), BC1-style 4096^2
texture, CTF_MODE_COLLAB with the C+ fallback, per-pixel uv + fp16 Jacobian in,
RGBA fp32 + per-wave records out.  One step = one ctf_filter_batch call over
the rank's share of the 64 frames.  Inputs are resident in HBM before timing;
the batch (17 GB of I/O) is far larger than L2, so no L2 flush is needed
between steps.  Multi-GPU: the path shards with no data
exchange (waves never read another wave's pixels).  Default
--split frames: rank g filters frames [g*64/G, (g+1)*64/G) of the fixed batch
(strong scaling, RNG frame indices = global frame numbers, so the results equal
the 1-GPU run bit for bit); --split strip: every rank filters its wave-row
strip of all 64 frames (ctf_params.row0); --split weak: every rank its own 64
frames.  NCCL carries only the max-over-ranks time and one all_gather of
statistics, reduced in rank order (paper_2506_17770_b200.dist).

At N = 1 the line also carries "configs": the other §8 configurations
(1: 64x64 launch latency, 2: 1080p, 3: 4K latent-MLP COLLAB vs 4-tap,
4: 4K mixed minification with every fallback), each timed on the device.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference ...                      # CPU oracle arm
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "4K filtered Gpix/s per B200 (1/2/4/8 GPUs); texel evals/pixel; error vs bilinear"
UNIT = "Gpix/s"
# the timed ABI call: BC1 COLLAB runs the lean exact kernel, then the wide-window kernel (32 x 32
# bitmap windows) and the third kernel (64 x 64 windows, the sort-based general path beyond)
# over the waves it marked (fallback / partial or wider windows); the roofline times the whole call
KERNEL_NAME = "ctf_collab_lean_kernel + 2 x ctf_collab_rest_kernel (one ctf_filter_batch call)"
MODES = {"collab": 3, "4tap": 0, "stf": 1, "wc": 2}
FALLBACKS = {"stf": 0, "wc": 1, "c": 2, "cplus": 3}
MLP_FMA_PER_EVAL = 32 * 12 + 32 * 32 + 4 * 32   # 1536 FMA per latent-MLP texel (R-10)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=64, help="frames in the batch (per rank with --split weak)")
    ap.add_argument("--split", choices=["frames", "strip", "weak"], default="frames",
                    help="multi-GPU partition (SURVEY §8(e)): frames = contiguous frame blocks of the fixed "
                         "batch (strong), strip = wave-row strips of every frame (strong), weak = every rank "
                         "its own batch of --frames frames")
    ap.add_argument("--width", type=int, default=3840)
    ap.add_argument("--height", type=int, default=2160)
    ap.add_argument("--tex", type=int, default=4096)
    ap.add_argument("--mode", choices=list(MODES), default="collab")
    ap.add_argument("--fallback", choices=list(FALLBACKS), default="cplus")
    ap.add_argument("--no-grad", action="store_true")
    ap.add_argument("--e2e-frames", type=int, default=32)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=1, help="frames per host-pipeline chunk (copy granularity)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other §8 configurations")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--profile-launches", type=int, default=0,
                    help="(for ncu) run this many launches after warmup, no timing/json")
    ap.add_argument("--profile-config3", type=int, default=0,
                    help="(for ncu) run this many config-3 latent-MLP COLLAB launches and exit")
    return ap.parse_args()


# --------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "power_w_max": max(power) if power else None, "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(frames: int, wf: int, hf: int):
    """dram bytes per launch of the dominant kernel, scaled from the committed ncu --set full capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        per_px = d["dram_bytes_per_launch"] / (d["frames"] * d["width"] * d["height"])
        return per_px * frames * wf * hf
    except Exception:
        return None


def ncu_issue(frames: int, wf: int, hf: int):
    """warp instructions per call of the timed kernels, scaled per pixel from the committed ncu
    --set full capture of one bench step (profiles/ncu_traffic.json), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d["warp_inst_per_launch"] / (d["frames"] * d["width"] * d["height"]) * frames * wf * hf
    except Exception:
        return None


def roofline_line(achieved, peak, traffic, issue, k_ms, bytes_per_launch, peak_src) -> dict:
    """frac = max(HBM fraction, issue fraction); `bound` names the larger one and
    the top-level achieved / peak / unit are its figures; both rooflines are kept."""
    hbm = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src}
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": KERNEL_NAME, "kernel_ms": k_ms, "kernel_ms_stat": "median",
         "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src, "hbm": hbm, "issue": issue}
    if issue is not None and issue["frac"] > hbm["frac"]:
        r.update(bound="issue", achieved=issue["achieved"], peak=issue["peak"], unit=issue["unit"], frac=issue["frac"])
    return r


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_check(oracle, tex_np, uv_t, g_t, out_t, rec_t, mode, fb, seed, frame_index, threads=None):
    """Time the CPU oracle (as it stands) on the exact bytes the GPU filtered and compare: records
    bit for bit, colours max |GPU - oracle|.  threads: OpenMP threads for this call (None = all)."""
    uv_np = uv_t.cpu().numpy()
    g_np = None if g_t is None else g_t.cpu().numpy()
    prev = oracle.set_threads(threads) if threads else None
    t0 = time.perf_counter()
    o = oracle.filter_frame(tex_np, uv_np, g_np, mode, fb, 0, seed, frame_index, debug=False)
    secs = time.perf_counter() - t0
    if prev:
        oracle.set_threads(prev)
    rec_ok = bool(np.array_equal(rec_t.cpu().numpy().view(np.uint32), o["rec"]))
    err = float(np.abs(out_t.cpu().numpy().astype(np.float64) - o["out"]).max())
    return secs, rec_ok, err


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def time_launches(fn, reps: int, stream) -> float:
    """Mean device time (ms) of `reps` back-to-back calls, CUDA events on the launching stream."""
    import torch
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def time_graph(fn, calls: int, stream, replays: int = 10) -> float:
    """Device time (ms) per call of `calls` calls captured in one CUDA graph and replayed: the
    per-call cost without host launch overhead (the library enqueues only on the given stream,
    so its calls are capturable)."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(calls):
                fn(s)
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(replays):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (replays * calls)


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synthetic
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
    oracle.build_oracle()
    blocks = synthetic.bc1_texture(args.tex, args.tex, args.seed, "image")
    mode, fb = MODES[args.mode], FALLBACKS[args.fallback]
    tex = {"format": 1, "width": args.tex, "height": args.tex, "bc1": blocks}
    # each step: one full 4K frame of the camera path (a bounded sample of the 64-frame batch)
    times = []
    for s in range(args.warmup + args.steps):
        f = (s * 7) % 64
        uv, g = synthetic.camera_path_frame(f, args.width, args.height, args.tex, args.tex)
        if args.no_grad:
            g = None
        t0 = time.perf_counter()
        oracle.filter_frame(tex, uv, g, mode, fb, 0, args.seed, f, debug=False)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = args.width * args.height / (ms / 1000.0) / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", cpu_cores()))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config5: camera-path 4K frames, BC1 4096^2, COLLAB(C+)",
                       "frames_per_step": 1, "width": args.width, "height": args.height, "tex": args.tex,
                       "mode": args.mode, "fallback": args.fallback, "grad": not args.no_grad},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "one full 4K camera-path frame per step (frames 7s mod 64)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- other §8 configs
def other_configs(ctf, torch, dev, stream, seed: int, peak_gbs: float, sm_mhz: float, cpu: bool = True) -> dict:
    """Configs 1-4 of BASELINE.json, each timed on the device (rank 0, N = 1); with `cpu`, the
    CPU oracle (as it stands, all host cores; config 2 also on one core) filters the same bytes,
    and its records / colours are compared with the GPU's (SURVEY §8(d) oracle baseline)."""
    import synthetic
    res = {}
    oracle = None
    if cpu:
        import oracle
        oracle.build_oracle()

    def cpu_leg(key, tex_np, uv, g, out, rec, mode, fb, threads=None):
        if oracle is None:
            return
        secs, rec_ok, err = oracle_check(oracle, tex_np, uv, g, out, rec, mode, fb, seed, 0, threads)
        px = uv.shape[0] * uv.shape[1]
        tag = "oracle_1thread" if threads == 1 else "oracle"
        res[key][tag] = {"ms_per_frame": secs * 1e3, "mpix_s": px / secs / 1e6,
                         "threads": threads or cpu_cores(), "records_equal_gpu": rec_ok, "max_abs_err_vs_gpu": err}
    fp32_peak_tflops = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12   # FFMA issue peak at max SM clock

    last = {}

    def run(tex, uv, g, mode, fb, reps):
        out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device=dev)
        rec = torch.empty(((uv.shape[0] + 3) // 4, (uv.shape[1] + 7) // 8), dtype=torch.int32, device=dev)
        ms = time_launches(lambda: ctf.filter_frame(tex, uv, g, mode, fb, 0, seed, 0, out=out, rec=rec,
                                                    stream=stream), reps, stream)
        st = ctf.stats(rec, uv.shape[1], uv.shape[0], 1, stream=stream)
        last["rec"] = rec
        return ms, st, out

    def graph_timing(tex, uv, g, wf, hf, calls):
        """single-frame calls back to back in a CUDA graph (device time per call, no host
        launch overhead): the library's one-launch fused path and the separate passes"""
        out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device=dev)
        rec = torch.empty(((uv.shape[0] + 3) // 4, (uv.shape[1] + 7) // 8), dtype=torch.int32, device=dev)
        ws = ctf.workspace_for(tex, 3, 0, wf, hf, 1, dev)
        r = {}
        for key, fl in (("graph_us_per_call", 0), ("graph_us_per_call_separate_passes", ctf.FLAG_SEPARATE_PASSES)):
            ms_g = time_graph(lambda s: ctf.filter_frame(tex, uv, g, 3, 3, fl, seed, 0, out=out, rec=rec, workspace=ws,
                                                         stream=s), calls, stream)
            r[key] = ms_g * 1e3
        r["graph_gpix_s"] = wf * hf / (r["graph_us_per_call"] / 1e6) / 1e9
        r["launches_per_call"] = ctf.launches_per_call(1, 3, 0, 1, False, wf=wf, hf=hf)
        return r

    def entry(wf, hf, ms, st, nbytes=None):
        e = {"ms": ms, "gpix_s": wf * hf / (ms / 1e3) / 1e9,
             "texel_evals_per_px": st["texel_evals"] / max(1, st["pixels_active"]),
             "exact_wave_frac": st["waves_exact"] / max(1, st["waves_live"])}
        if nbytes is not None:
            e["hbm_frac"] = nbytes / (ms / 1e3) / 1e9 / peak_gbs
        return e

    # config 1: 64x64 frame, 32^2 BC1, uniform 4x — launch-latency bound
    b1 = synthetic.bc1_texture(32, 32, seed, "image")
    t1 = ctf.Texture.bc1(b1, 32, 32, device=dev)
    uv, g = synthetic.rotated_quad(64, 64, 32, 32, 4.0, 30.0)
    uv, g = torch.from_numpy(uv).to(dev), torch.from_numpy(g).to(dev)
    ms, st, out = run(t1, uv, g, 3, 3, 200)
    res["1_64x64_bc1_m4"] = dict(entry(64, 64, ms, st), us_per_launch=ms * 1e3)
    res["1_64x64_bc1_m4"].update(graph_timing(t1, uv, g, 64, 64, 50))
    cpu_leg("1_64x64_bc1_m4", {"format": 1, "width": 32, "height": 32, "bc1": b1}, uv, g, out, last["rec"], 3, 3)

    # config 2: 1080p, 2048^2 BC1, perspective plane (m ~0.9-9.4, mean 4.3)
    b2 = synthetic.bc1_texture(2048, 2048, seed, "image")
    t2 = ctf.Texture.bc1(b2, 2048, 2048, device=dev)
    uv, g = synthetic.perspective_plane_torch(1920, 1080, 2048, 2048, synthetic.PLANE_C2, device=dev)
    ms, st, out = run(t2, uv, g, 3, 3, 50)
    res["2_1080p_bc1_collab_cplus"] = entry(1920, 1080, ms, st, 1920 * 1080 * 32)
    res["2_1080p_bc1_collab_cplus"].update(graph_timing(t2, uv, g, 1920, 1080, 50))
    tex2 = {"format": 1, "width": 2048, "height": 2048, "bc1": b2}
    cpu_leg("2_1080p_bc1_collab_cplus", tex2, uv, g, out, last["rec"], 3, 3)
    cpu_leg("2_1080p_bc1_collab_cplus", tex2, uv, g, out, last["rec"], 3, 3, threads=1)

    # config 3: 4K, 4096^2 latent-MLP texture, COLLAB vs 4-tap (FP32-pipe bound)
    lat3, mlp3 = synthetic.latent_texture(4096, 4096, seed), synthetic.mlp_weights(seed + 1)
    t3 = ctf.Texture.latent_mlp(lat3, mlp3, 4096, 4096, device=dev)
    uv, g = synthetic.perspective_plane_torch(3840, 2160, 4096, 4096, synthetic.PLANE_C2, device=dev)
    for name, mode in (("collab_cplus", 3), ("4tap", 0)):
        ms, st, out = run(t3, uv, g, mode, 3, 10 if mode == 3 else 3)
        e = entry(3840, 2160, ms, st)
        fl = st["texel_evals"] * MLP_FMA_PER_EVAL * 2
        e["mlp_tflops"] = fl / (ms / 1e3) / 1e12
        e["fp32_frac"] = e["mlp_tflops"] / fp32_peak_tflops
        res[f"3_4k_latent_mlp_{name}"] = e
        if mode == 3:
            collab_out = out
            cpu_leg(f"3_4k_latent_mlp_{name}", {"format": 2, "width": 4096, "height": 4096, "latent": lat3, "mlp": mlp3},
                    uv, g, out, last["rec"], 3, 3)
        else:
            d = (collab_out.double() - out.double())
            res["3_4k_latent_mlp_collab_cplus"]["max_abs_err_vs_4tap"] = float(d.abs().max())
    # config 4: 4K, 4096^2 BC1, grazing plane (horizon, minified waves), every fallback
    b4 = synthetic.bc1_texture(4096, 4096, seed, "image")
    t4 = ctf.Texture.bc1(b4, 4096, 4096, device=dev)
    uv, g = synthetic.perspective_plane_torch(3840, 2160, 4096, 4096, synthetic.PLANE_C4, device=dev)
    _, _, ref = run(t4, uv, g, 0, 0, 1)
    ref = ref.clone()
    for name, fb in FALLBACKS.items():
        ms, st, out = run(t4, uv, g, 3, fb, 10)
        e = entry(3840, 2160, ms, st, 3840 * 2160 * 32)
        e["fallback_wave_frac"] = st["waves_fallback"] / max(1, st["waves_live"])
        cov = ~torch.isnan(uv[..., 0])
        err = (out - ref)[cov].double()
        mse = float((err * err).mean())
        e["psnr_vs_bilinear_db"] = 10 * float(np.log10(1.0 / mse)) if mse > 0 else float("inf")
        res[f"4_4k_mixed_bc1_collab_{name}"] = e
        if name == "cplus":
            cpu_leg(f"4_4k_mixed_bc1_collab_{name}", {"format": 1, "width": 4096, "height": 4096, "bc1": b4},
                    uv, g, out, last["rec"], 3, fb)
    # the paper's three exact methods on the same grazing scene, C+ fallback (Fig. 4 / Fig. 7 shape)
    for name, mode in (("list", 3), ("box", 4), ("mask16", 5), ("mask11", 6)):
        ms, st, out = run(t4, uv, g, mode, 3, 10)
        e = entry(3840, 2160, ms, st, 3840 * 2160 * 32)
        cov = ~torch.isnan(uv[..., 0])
        err = (out - ref)[cov].double()
        mse = float((err * err).mean())
        e["psnr_vs_bilinear_db"] = 10 * float(np.log10(1.0 / mse)) if mse > 0 else float("inf")
        res[f"4_4k_mixed_bc1_method_{name}_cplus"] = e
    # bicubic filters (§5.4, Fig. 13): 4K perspective plane of config 3 with the BC1 texture
    uv, g = synthetic.perspective_plane_torch(3840, 2160, 4096, 4096, synthetic.PLANE_C2, device=dev)
    cov = ~torch.isnan(uv[..., 0])
    # (BC1: both filters; the latent-MLP texture of config 3: Catmull-Rom, where the evaluation
    # saving — ~0.8 instead of 16 evaluations per pixel — is the whole cost)
    for fname, filt, tex_b, variants in (
            ("bspline", 1, t4, None), ("catmull_rom", 2, t4, None),
            ("catmull_rom_latent_mlp", 2, t3, (("full16", 0, 0, 1), ("list_cplus_e2", 3, 3, 2)))):
        def runb(mode, fb, E, reps):
            out = torch.empty(uv.shape[:-1] + (4,), dtype=torch.float32, device=dev)
            rec = torch.empty(((uv.shape[0] + 3) // 4, (uv.shape[1] + 7) // 8), dtype=torch.int32, device=dev)
            ms = time_launches(lambda: ctf.filter_frame(tex_b, uv, g, mode, fb, 0, seed, 0, out=out, rec=rec,
                                                        stream=stream, filter=filt, max_evals=E), reps, stream)
            return ms, ctf.stats(rec, uv.shape[1], uv.shape[0], 1, stream=stream), out
        _, _, full = runb(0, 0, 1, 1)
        full = full.clone()
        for name, mode, fb, E in variants or (("full16", 0, 0, 1), ("stf_positivized", 1, 0, 1),
                                              ("list_cplus_e1", 3, 3, 1), ("list_cplus_e2", 3, 3, 2),
                                              ("box_cplus_e2", 4, 3, 2)):
            ms, st, out = runb(mode, fb, E, (1 if tex_b is t3 else 3) if mode == 0 else (3 if tex_b is t3 else 10))
            e = entry(3840, 2160, ms, st, 3840 * 2160 * 32)
            err = (out - full)[cov].double()
            mse = float((err * err).mean())
            e["psnr_vs_full_filter_db"] = 10 * float(np.log10(1.0 / mse)) if mse > 0 else float("inf")
            e["max_evals_per_lane"] = st["max_evals_per_lane"]
            res[f"6_4k_bicubic_{fname}_{name}"] = e
    return res


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as tdist

    import synthetic
    from paper_2506_17770_b200 import build as pbuild
    from paper_2506_17770_b200 import dist as cdist
    import paper_2506_17770_b200.ctf as ctf

    ws, rank, local = dist_env()
    if ws > 1:
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    pbuild.build()
    ctf.load_library()
    if args.profile_config3:
        t3 = ctf.Texture.latent_mlp(synthetic.latent_texture(4096, 4096, args.seed),
                                    synthetic.mlp_weights(args.seed + 1), 4096, 4096, device=dev)
        u3, g3 = synthetic.perspective_plane_torch(3840, 2160, 4096, 4096, synthetic.PLANE_C2, device=dev)
        for _ in range(args.profile_config3):
            ctf.filter_frame(t3, u3, g3, 3, 3, 0, args.seed, 0)
        torch.cuda.synchronize()
        return 0

    Wf, Hf, T = args.width, args.height, args.tex
    mode, fb = MODES[args.mode], FALLBACKS[args.fallback]
    blocks = synthetic.bc1_texture(T, T, args.seed, "image")
    tex = ctf.Texture.bc1(blocks, T, T, device=dev)   # every rank builds the same texture from the seed
    # this rank's share of the work; each rank generates only its own inputs
    row0, Hr = 0, Hf
    if args.split == "weak":
        path_frames, frame_base = cdist.weak_frames(args.frames, rank)
        F_total = ws * args.frames
    else:
        F_total = args.frames
        if args.split == "frames":
            shard = cdist.frame_shard(F_total, ws, rank)
            path_frames, frame_base = list(shard), shard.start
        else:
            path_frames, frame_base = list(range(F_total)), 0
            row0, Hr = cdist.strip_shard(Hf, ws, rank)
    F = len(path_frames)
    uv = torch.empty((F, Hr, Wf, 2), dtype=torch.float32, device=dev)
    grad = None if args.no_grad else torch.empty((F, Hr, Wf, 4), dtype=torch.float16, device=dev)
    for i, f in enumerate(path_frames):
        u, g = synthetic.camera_path_frame_torch(f, Wf, Hf, T, T, device=dev)
        uv[i].copy_(u[row0:row0 + Hr])
        if grad is not None:
            grad[i].copy_(g[row0:row0 + Hr])
        del u, g
    out = torch.empty((F, Hr, Wf, 4), dtype=torch.float32, device=dev)
    nwy, nwx = (Hr + 3) // 4, (Wf + 7) // 8
    rec = torch.empty((F, nwy, nwx), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    wspace = ctf.workspace_for(tex, mode, 0, Wf, Hr, F, dev)   # work lists (ctf_params.workspace_dev)

    def step():
        ctf.filter_batch(tex, uv, grad, mode, fb, 0, args.seed, frame_base, out=out, rec=rec, stream=stream,
                         workspace=wspace, row0=row0)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if args.profile_launches:
        for _ in range(args.profile_launches):
            step()
        torch.cuda.synchronize()
        return 0

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ws > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    clk = clocks.stop()
    elapsed_ms = cdist.max_over_ranks(t0.elapsed_time(t1), device=dev)
    kernel_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_per_step = elapsed_ms / args.steps
    value = F_total * Wf * Hf / (ms_per_step / 1e3) / 1e9   # whole job: every rank's pixels / max-over-ranks time

    # roofline of the dominant (only) kernel: algorithmic bytes per launch / mean launch time
    nwaves = nwy * nwx
    bytes_per_launch = F * (Wf * Hr * (8 + (0 if grad is None else 8) + 16) + nwaves * 4)
    k_ms = statistics.median(kernel_ms)   # the median over the timed steps
    achieved = bytes_per_launch / (k_ms / 1e3) / 1e9
    peak, sm_mhz, peak_src = measured_peaks()
    traffic = ncu_traffic(F, Wf, Hr)
    # the issue roofline (§8(d)): warp instructions per call (ncu capture) / (4 schedulers x SMs x clock)
    inst = ncu_issue(F, Wf, Hr)
    clk_mhz = clk.get("sm_mhz") or sm_mhz
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    issue = None if inst is None else {
        "achieved": inst / (k_ms / 1e3) / 1e9, "peak": 4 * n_sms * clk_mhz * 1e6 / 1e9, "unit": "Gwarp-inst/s",
        "frac": inst / (k_ms / 1e3) / (4 * n_sms * clk_mhz * 1e6), "warp_inst_per_call": inst,
        "source": "profiles/ncu_traffic.json (ncu --set full of one bench step), SM clock = median under load"}

    # quality + statistics (off the timed path): 4-tap reference, ctf_stats, NCCL all_gather
    ref = torch.empty_like(out)
    ctf.filter_batch(tex, uv, grad, 0, 0, 0, args.seed, frame_base, out=ref, rec=torch.empty_like(rec), stream=stream,
                     row0=row0)
    per_frame = []   # per-frame records, reduced in global frame order on every rank (dist.reduce_frame_stats)
    for i in range(F):
        st = ctf.stats(rec[i], Wf, Hr, 1, out[i], ref[i], stream=stream)
        st["frame"], st["row0"] = frame_base + i, row0
        per_frame.append(st)
    del ref
    tot = cdist.reduce_frame_stats(per_frame)
    mse = tot["sum_sq_err"] / max(1, 4 * tot["pixels_active"])
    quality = {
        "texel_evals_per_px": tot["texel_evals"] / max(1, tot["pixels_active"]),
        "texel_evals_per_px_magnified_waves": tot["texel_evals_in_magnified_waves"] / max(1, tot["pixels_in_magnified_waves"]),
        "exact_wave_frac": tot["waves_exact"] / max(1, tot["waves_live"]),
        "magnified_wave_frac": tot["waves_magnified"] / max(1, tot["waves_live"]),
        "max_unique_per_wave": tot["max_unique_per_wave"],
        "max_evals_per_lane": tot["max_evals_per_lane"],
        "psnr_vs_bilinear_db": (10.0 * np.log10(1.0 / mse)) if mse > 0 else float("inf"),
        "max_abs_err_vs_bilinear": tot["max_abs_err"],
    }

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        E = min(args.e2e_frames, F)
        uv_h = uv[:E].cpu().pin_memory()
        g_h = None if grad is None else grad[:E].cpu().pin_memory()
        out_h = torch.empty((E, Hr, Wf, 4), dtype=torch.float32).pin_memory()
        rec_h = torch.empty((E, nwy, nwx), dtype=torch.int32).pin_memory()
        chunk = max(1, args.e2e_chunk)  # frames per chunk: the copy engines overlap H2D(c+1), kernel(c), D2H(c-1)
        pipe = ctf.HostPipeline(Wf, Hr, chunk, grad is not None, device=dev)
        pipe.run(tex, uv_h, g_h, out_h, rec_h, mode, fb, 0, args.seed, frame_base, stream=stream, row0=row0)  # warm
        if ws > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.e2e_steps):
            pipe.run(tex, uv_h, g_h, out_h, rec_h, mode, fb, 0, args.seed, frame_base, stream=stream, row0=row0)
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = cdist.max_over_ranks(a0.elapsed_time(a1) / args.e2e_steps, device=dev)
        h2d_b = E * Wf * Hr * (8 + (0 if grad is None else 8))
        d2h_b = E * (Wf * Hr * 16 + nwaves * 4)
        # the link bound: each direction's pinned-copy bandwidth, measured alone
        bw = {}
        for name, (src, dst) in {"h2d": (out_h, out), "d2h": (out, out_h)}.items():
            n = min(src[0].numel(), dst[0].numel()) * 4
            s_, d_ = src[0].view(-1), dst[0].view(-1)
            d_.copy_(s_, non_blocking=True)
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(5):
                d_.copy_(s_, non_blocking=True)
            b1.record(stream)
            torch.cuda.synchronize()
            bw[name] = 5 * n / (b0.elapsed_time(b1) / 1e3) / 1e9
        link_ms = max(h2d_b / bw["h2d"], d2h_b / bw["d2h"]) / 1e6
        e2e_px = cdist.sum_over_ranks(E * Wf * Hr, device=dev)
        e2e = {"value": e2e_px / (e_ms / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "frames_per_step": E,
               "chunk_frames": chunk, "ms_per_step": e_ms,
               "pcie_gbs": {"h2d": bw["h2d"], "d2h": bw["d2h"]},
               "link_bound_ms_per_step": link_ms, "link_frac": link_ms / e_ms,
               "api": "ctf_filter_frames_host (pinned host buffers)"}
        del uv_h, g_h, out_h, rec_h, pipe

    configs = None
    if rank == 0 and ws == 1 and not args.no_configs:
        configs = other_configs(ctf, torch, dev, stream, args.seed, peak, sm_mhz, cpu=not args.no_cpu)

    # CPU oracle baseline on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
        import oracle
        oracle.build_oracle()
        otex = {"format": 1, "width": T, "height": T, "bc1": blocks}
        px, secs, nfr = 0, 0.0, 0
        rec_ok, worst = True, 0.0
        order = list(range(0, F, 8)) + [f for f in range(F) if f % 8]
        while secs < args.cpu_seconds and nfr < F:
            i = order[nfr]
            dt, ok, err = oracle_check(oracle, otex, uv[i], None if grad is None else grad[i], out[i], rec[i], mode, fb,
                                       args.seed, frame_base + i)
            secs += dt
            rec_ok &= ok
            worst = max(worst, err)
            px += Wf * Hr
            nfr += 1
        cpu = {"value": px / secs / 1e9, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{nfr} full 4K frames of the batch (every 8th first), {secs:.1f} s of oracle time",
               "parity_vs_gpu": {"frames": nfr, "records_equal": rec_ok, "max_abs_err": worst, "tolerance": 1e-5}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "ms_per_step_median": statistics.median(kernel_ms), "ms_per_step_min": min(kernel_ms),
            "scaling": "weak" if args.split == "weak" else "strong",
            "per_gpu_value": value / ws,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config5: 64-frame 4K camera path over a perspective plane, BC1 4096^2, "
                                   "COLLAB + C+ fallback, uv f32x2 + grad f16x4 in, RGBA f32 out",
                       "frames_per_step": F_total, "frames_per_rank": F, "rows_per_rank": Hr,
                       "width": Wf, "height": Hf, "tex": T, "mode": args.mode,
                       "fallback": args.fallback, "grad": grad is not None,
                       "l2": "inputs (17 GB/step) >> L2, no flush needed",
                       "parallelism": {"frames": f"frame blocks of the {F_total}-frame batch x{ws} (strong)",
                                       "strip": f"wave-row strips of every frame x{ws} (strong)",
                                       "weak": f"{args.frames} frames per rank x{ws} (weak)"}[args.split]},
            "roofline": roofline_line(achieved, peak, traffic, issue, k_ms, bytes_per_launch, peak_src),
            "quality": quality,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * ctf.launches_per_call(1, mode, 0, F, True, workspace=True, wf=Wf, hf=Hr),
            "clocks": clk,
            "configs": configs,
        }
        print(json.dumps(line))
    if ws > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
