"""ctypes wrapper + plain-numpy stats for the C oracle (test infrastructure only).

Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SRC = HERE / "ctf_oracle.c"
ORACLE_SO = HERE / "libctf_oracle.so"

FMT_BC1, FMT_LATENT_MLP = 1, 2
M_4TAP, M_STF, M_WC, M_COLLAB, M_BOX, M_MASK16, M_MASK11 = 0, 1, 2, 3, 4, 5, 6
FB_STF, FB_WC, FB_C, FB_CPLUS = 0, 1, 2, 3
FL_DEBUG, FL_FORCE_FALLBACK = 1, 2
FILTER_BILINEAR, FILTER_BSPLINE, FILTER_CATMULL_ROM = 0, 1, 2

_lib = None


def build_oracle(force: bool = False) -> Path:
    if force or not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < ORACLE_SRC.stat().st_mtime:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", str(ORACLE_SO), str(ORACLE_SRC), "-lm"]
        subprocess.run(cmd, check=True)
    return ORACLE_SO


def load_oracle():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(str(ORACLE_SO))
        P = ctypes.c_void_p
        i32, u32, u64 = ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
        lib.oracle_filter_frame.argtypes = [i32, i32, i32, P, P, P, P, P, i32, i32,
                                            i32, i32, u32, u64, u32, P, P, P, P]
        lib.oracle_filter_frame.restype = i32
        lib.oracle_filter_waves.argtypes = [i32, i32, i32, P, P, P, P, P, i32, i32,
                                            i32, i32, u32, u64, u32, P, i32, P, P, P, P]
        lib.oracle_filter_waves.restype = i32
        lib.oracle_filter_frame2.argtypes = [i32, i32, i32, P, P, P, P, P, i32, i32,
                                             i32, i32, u32, u64, u32, i32, i32, P, P, P, P]
        lib.oracle_filter_frame2.restype = i32
        lib.oracle_filter_waves2.argtypes = [i32, i32, i32, P, P, P, P, P, i32, i32,
                                             i32, i32, u32, u64, u32, i32, i32, P, i32, P, P, P, P]
        lib.oracle_filter_waves2.restype = i32
        lib.oracle_cubic_weights.argtypes = [i32, ctypes.c_float, P]
        lib.oracle_philox4x32_10.argtypes = [P, P, P]
        lib.oracle_bc1_texel.argtypes = [P, i32, i32, i32, P]
        lib.oracle_mlp_texel.argtypes = [P, P, i32, i32, i32, i32, P]
        lib.oracle_footprint.argtypes = [ctypes.c_float, ctypes.c_float, i32, i32, P, P]
        lib.oracle_h.argtypes = [u32, u32]
        lib.oracle_h.restype = i32
        lib.oracle_h_inv.argtypes = [i32, u32]
        lib.oracle_h_inv.restype = i32
        lib.oracle_eq2.argtypes = [i32, i32, i32]
        lib.oracle_eq2.restype = i32
        lib.oracle_unique_count.argtypes = [P, i32]
        lib.oracle_unique_count.restype = i32
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_set_threads.restype = i32
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _tex_args(tex):
    fmt = tex["format"]
    if fmt == FMT_BC1:
        return fmt, tex["width"], tex["height"], np.ascontiguousarray(tex["bc1"], np.uint8), None, None
    lat = np.ascontiguousarray(tex["latent"], np.float16).view(np.uint16)
    return fmt, tex["width"], tex["height"], None, lat, np.ascontiguousarray(tex["mlp"], np.float32)


def filter_frame(tex: dict, uv: np.ndarray, grad: np.ndarray | None, mode: int, fallback: int = FB_CPLUS,
                 flags: int = 0, seed: int = 0, frame_index: int = 0, debug: bool = True,
                 filter: int = FILTER_BILINEAR, max_evals: int = 1):
    """Run the oracle on one frame.  Returns dict(out fp64 [Hf][Wf][4], rec, produced_id, selection)."""
    lib = load_oracle()
    hf, wf = uv.shape[:2]
    uv = np.ascontiguousarray(uv, np.float32)
    g = None if grad is None else np.ascontiguousarray(grad, np.float16).view(np.uint16)
    fmt, W, H, bc1, lat, mlp = _tex_args(tex)
    out = np.zeros((hf, wf, 4), np.float64)
    rec = np.zeros(((hf + 3) // 4, (wf + 7) // 8), np.uint32)
    pid = np.zeros((hf, wf), np.uint32) if debug else None
    sel = np.zeros((hf, wf), np.uint32) if debug else None
    rc = lib.oracle_filter_frame2(fmt, W, H, _ptr(bc1), _ptr(lat), _ptr(mlp), _ptr(uv), _ptr(g), wf, hf,
                                  mode, fallback, flags, seed, frame_index, filter, max_evals,
                                  _ptr(out), _ptr(rec), _ptr(pid), _ptr(sel))
    if rc != 0:
        raise ValueError("oracle_filter_frame: invalid arguments")
    return {"out": out, "rec": rec, "produced_id": pid, "selection": sel}


def filter_waves(tex: dict, uv: np.ndarray, grad: np.ndarray | None, waves: np.ndarray, mode: int,
                 fallback: int = FB_CPLUS, flags: int = 0, seed: int = 0, frame_index: int = 0,
                 filter: int = FILTER_BILINEAR, max_evals: int = 1):
    """Oracle restricted to the listed wave indices (wy * nwx + wx); other outputs stay 0."""
    lib = load_oracle()
    hf, wf = uv.shape[:2]
    uv = np.ascontiguousarray(uv, np.float32)
    g = None if grad is None else np.ascontiguousarray(grad, np.float16).view(np.uint16)
    fmt, W, H, bc1, lat, mlp = _tex_args(tex)
    waves = np.ascontiguousarray(waves, np.int32)
    out = np.zeros((hf, wf, 4), np.float64)
    rec = np.zeros(((hf + 3) // 4, (wf + 7) // 8), np.uint32)
    pid = np.zeros((hf, wf), np.uint32)
    sel = np.zeros((hf, wf), np.uint32)
    rc = lib.oracle_filter_waves2(fmt, W, H, _ptr(bc1), _ptr(lat), _ptr(mlp), _ptr(uv), _ptr(g), wf, hf,
                                  mode, fallback, flags, seed, frame_index, filter, max_evals,
                                  _ptr(waves), len(waves), _ptr(out), _ptr(rec), _ptr(pid), _ptr(sel))
    if rc != 0:
        raise ValueError("oracle_filter_waves: invalid arguments")
    return {"out": out, "rec": rec, "produced_id": pid, "selection": sel}


def cubic_weights(filter: int, s: float) -> np.ndarray:
    """fp32 tap weights of the B-spline (1) / Catmull-Rom (2) kernel at fraction s (R-25)."""
    lib = load_oracle()
    w = np.zeros(4, np.float32)
    lib.oracle_cubic_weights(filter, ctypes.c_float(s), _ptr(w))
    return w


def decode_record(rec: np.ndarray) -> dict:
    """Per-wave record fields (DESIGN.md / include/ctf.h layout)."""
    r = rec.astype(np.uint64)
    return {
        "evals": ((r & 0xFF) | (((r >> 27) & 0x7) << 8)).astype(np.int64),
        "n": ((r >> 8) & 0xFF).astype(np.int64),
        "a": ((r >> 16) & 0x3F).astype(np.int64),
        "path": ((r >> 22) & 0x7).astype(np.int64),
        "magnified": ((r >> 25) & 1).astype(np.int64),
        "partial": ((r >> 26) & 1).astype(np.int64),
    }


def frame_stats(rec: np.ndarray, out: np.ndarray | None = None, ref: np.ndarray | None = None,
                covered: np.ndarray | None = None) -> dict:
    """Plain-numpy frame totals from per-wave records (what ctf_stats must return)."""
    d = decode_record(rec.reshape(-1))
    live = d["a"] > 0
    mag = live & (d["magnified"] == 1)
    exact = live & (d["path"] == 0)
    fb = live & (d["path"] >= 1) & (d["path"] <= 4)
    hist = np.zeros(129, np.int64)
    nvalid = live & (d["n"] <= 128)
    np.add.at(hist, d["n"][nvalid], 1)
    st = {
        "waves_live": int(live.sum()),
        "waves_partial": int((live & (d["partial"] == 1)).sum()),
        "waves_exact": int(exact.sum()),
        "waves_fallback": int(fb.sum()),
        "waves_magnified": int(mag.sum()),
        "pixels_active": int(d["a"].sum()),
        "pixels_in_magnified_waves": int(d["a"][mag].sum()),
        "texel_evals": int(d["evals"].sum()),
        "texel_evals_in_magnified_waves": int(d["evals"][mag].sum()),
        "max_evals_per_lane": 0,
        "max_unique_per_wave": int(d["n"][nvalid].max()) if nvalid.any() else 0,
        "unique_hist": hist,
    }
    # evals per lane = ceil(evals / a): exact path and fallbacks 1 (2 with max_evals = 2 or
    # positivized STF), 4TAP 4 (16 for bicubic)
    per_lane = (d["evals"] + np.maximum(d["a"], 1) - 1) // np.maximum(d["a"], 1)
    st["max_evals_per_lane"] = int(per_lane[live].max()) if live.any() else 0
    if out is not None and ref is not None:
        o = out.astype(np.float64).reshape(-1, 4)
        r_ = ref.astype(np.float64).reshape(-1, 4)
        if covered is None:
            covered = np.ones(o.shape[0], bool)
        covered = covered.reshape(-1)
        e = (o - r_)[covered]
        st["sum_sq_err"] = float((e * e).sum())
        st["max_abs_err"] = float(np.abs(e).max()) if e.size else 0.0
        st["err_pixels"] = int(covered.sum())
    return st


# ---- small exported helpers for the pins ---------------------------------------------------

def philox4x32_10(ctr, key):
    lib = load_oracle()
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib.oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def bc1_texel(blocks: np.ndarray, width: int, x: int, y: int):
    lib = load_oracle()
    b = np.ascontiguousarray(blocks, np.uint8)
    o = np.zeros(4, np.uint8)
    lib.oracle_bc1_texel(_ptr(b), width, x, y, _ptr(o))
    return o


def mlp_texel(latent: np.ndarray, mlp: np.ndarray, width: int, height: int, x: int, y: int):
    lib = load_oracle()
    lat = np.ascontiguousarray(latent, np.float16).view(np.uint16)
    w = np.ascontiguousarray(mlp, np.float32)
    o = np.zeros(4, np.float64)
    lib.oracle_mlp_texel(_ptr(lat), _ptr(w), width, height, x, y, _ptr(o))
    return o


def footprint(u: float, v: float, width: int, height: int):
    lib = load_oracle()
    ids = np.zeros(4, np.uint32)
    st = np.zeros(2, np.float32)
    lib.oracle_footprint(u, v, width, height, _ptr(ids), _ptr(st))
    return ids, st


def h(i: int, mask: int) -> int:
    return load_oracle().oracle_h(i, mask)


def h_inv(t: int, mask: int) -> int:
    return load_oracle().oracle_h_inv(t, mask)


def eq2(c: int, n: int, a: int = 32) -> int:
    return load_oracle().oracle_eq2(c, n, a)


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's wave loops (0 = query); returns the previous count."""
    return load_oracle().oracle_set_threads(n)


def unique_count(ids) -> int:
    a = np.ascontiguousarray(ids, np.uint32)
    return load_oracle().oracle_unique_count(_ptr(a), len(a))


if os.environ.get("CTF_ORACLE_REBUILD"):
    build_oracle(force=True)
