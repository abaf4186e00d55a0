"""Thin ctypes binding of libctf.so (include/ctf.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI.  Tensors
are torch CUDA tensors (PyTorch supplies device memory and streams only); this
module never computes any part of the method and has no CPU fallback: if the
shared library is missing or a CUDA device is absent, calls raise.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import torch

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libctf.so"

CTF_OK, CTF_EINVAL, CTF_EUNSUPPORTED, CTF_EALIGN, CTF_ECUDA = 0, -1, -2, -3, -4
FMT_BC1, FMT_LATENT_MLP = 1, 2
MODE_4TAP, MODE_STF, MODE_WAVECOMM, MODE_COLLAB, MODE_BOX, MODE_MASK16, MODE_MASK11 = 0, 1, 2, 3, 4, 5, 6
FB_STF, FB_WAVECOMM, FB_C, FB_CPLUS = 0, 1, 2, 3
FLAG_DEBUG, FLAG_FORCE_FALLBACK, FLAG_SEPARATE_PASSES = 1, 2, 4
FILTER_BILINEAR, FILTER_BSPLINE, FILTER_CATMULL_ROM = 0, 1, 2
_STATUS = {0: "CTF_OK", -1: "CTF_EINVAL", -2: "CTF_EUNSUPPORTED", -3: "CTF_EALIGN", -4: "CTF_ECUDA"}


class CtfError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {_STATUS.get(code, code)}")
        self.code = code


class ctf_texture(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("addr", ctypes.c_int32), ("data_dev", ctypes.c_void_p), ("mlp_dev", ctypes.c_void_p),
                ("mlp_host", ctypes.c_void_p)]


class ctf_params(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("fallback", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("frame_index", ctypes.c_uint32), ("seed", ctypes.c_uint64), ("filter", ctypes.c_int32),
                ("max_evals", ctypes.c_int32), ("workspace_dev", ctypes.c_void_p), ("workspace_bytes", ctypes.c_uint64),
                ("row0", ctypes.c_int32), ("reserved_", ctypes.c_int32)]


class ctf_debug(ctypes.Structure):
    _fields_ = [("produced_id_dev", ctypes.c_void_p), ("selection_dev", ctypes.c_void_p),
                ("unread_dev", ctypes.c_void_p)]


class ctf_frame_stats(ctypes.Structure):
    _fields_ = [("waves_live", ctypes.c_uint64), ("waves_partial", ctypes.c_uint64),
                ("waves_exact", ctypes.c_uint64), ("waves_fallback", ctypes.c_uint64),
                ("waves_magnified", ctypes.c_uint64), ("pixels_active", ctypes.c_uint64),
                ("pixels_in_magnified_waves", ctypes.c_uint64), ("texel_evals", ctypes.c_uint64),
                ("texel_evals_in_magnified_waves", ctypes.c_uint64), ("max_evals_per_lane", ctypes.c_uint32),
                ("max_unique_per_wave", ctypes.c_uint32), ("unique_hist", ctypes.c_uint64 * 129),
                ("sum_sq_err", ctypes.c_double), ("max_abs_err", ctypes.c_float), ("pad_", ctypes.c_uint32),
                ("err_pixels", ctypes.c_uint64)]

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("unique_hist", "pad_")}
        d["unique_hist"] = list(self.unique_hist)
        return d


EXPORTS = ["ctf_filter_frame", "ctf_filter_batch", "ctf_stats", "ctf_host_workspace_bytes",
           "ctf_filter_frames_host", "ctf_filter_workspace_bytes", "ctf_launches_per_call", "ctf_abi_version"]

_lib = None


def load_library(path: Path | str | None = None):
    """Load libctf.so and declare the ABI.  Raises if the library is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(p))
    V, I32, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32
    PT, PP, PD = ctypes.POINTER(ctf_texture), ctypes.POINTER(ctf_params), ctypes.POINTER(ctf_debug)
    lib.ctf_filter_frame.argtypes = [PT, V, V, I32, I32, PP, V, V, PD, V]
    lib.ctf_filter_batch.argtypes = [PT, V, V, I32, I32, I32, PP, V, V, PD, V]
    lib.ctf_stats.argtypes = [V, I32, I32, I32, V, V, ctypes.POINTER(ctf_frame_stats), V]
    lib.ctf_host_workspace_bytes.argtypes = [I32, I32, I32, ctypes.c_int]
    lib.ctf_host_workspace_bytes.restype = ctypes.c_size_t
    lib.ctf_filter_workspace_bytes.argtypes = [I32, I32, I32]
    lib.ctf_filter_workspace_bytes.restype = ctypes.c_size_t
    lib.ctf_filter_frames_host.argtypes = [PT, V, V, I32, I32, I32, I32, PP, V, V, V, ctypes.c_size_t, V]
    lib.ctf_launches_per_call.argtypes = [I32, I32, I32, I32, I32, I32, ctypes.c_int]
    for fn in ("ctf_filter_frame", "ctf_filter_batch", "ctf_stats", "ctf_filter_frames_host",
               "ctf_launches_per_call", "ctf_abi_version"):
        getattr(lib, fn).restype = ctypes.c_int
    if path is None:
        _lib = lib
    return lib


def _check(fn: str, rc: int):
    if rc != CTF_OK:
        raise CtfError(fn, rc)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (the hot path has no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream: torch.cuda.Stream | None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Texture:
    """Device-resident texture (keeps the tensors alive) + its ctf_texture descriptor."""

    def __init__(self, fmt: int, width: int, height: int, data: torch.Tensor, mlp: torch.Tensor | None = None):
        self.fmt, self.width, self.height = fmt, width, height
        self.data, self.mlp = data, mlp
        # host copy of the MLP weights: passed by value into the kernel parameter block
        self.mlp_host = mlp.detach().cpu().contiguous() if mlp is not None else None
        self.desc = ctf_texture(fmt, width, height, 0, data.data_ptr(), mlp.data_ptr() if mlp is not None else None,
                                self.mlp_host.data_ptr() if self.mlp_host is not None else None)

    @staticmethod
    def bc1(blocks, width: int, height: int, device="cuda") -> "Texture":
        t = torch.as_tensor(blocks).to(device=device, dtype=torch.uint8).contiguous()
        return Texture(FMT_BC1, width, height, t)

    @staticmethod
    def latent_mlp(latent, mlp, width: int, height: int, device="cuda") -> "Texture":
        lat = torch.as_tensor(latent).to(device=device).contiguous()
        if lat.dtype != torch.float16:
            raise ValueError("latent grid must be float16")
        w = torch.as_tensor(mlp).to(device=device, dtype=torch.float32).contiguous()
        return Texture(FMT_LATENT_MLP, width, height, lat, w)


def launches_per_call(fmt: int, mode: int, filt: int = 0, frames: int = 1, batched: bool = True,
                      workspace: bool = False, wf: int = 3840, hf: int = 2160, separate: bool = False) -> int:
    """Kernel launches one filter call of `frames` wf x hf frames issues (ctf_launches_per_call)."""
    flags = int(batched) | (2 if workspace else 0) | (4 if separate else 0)
    n = load_library().ctf_launches_per_call(fmt, mode, filt, wf, hf, frames, flags)
    if n < 0:
        raise CtfError("ctf_launches_per_call", CTF_EINVAL)
    return n


def num_waves(wf: int, hf: int) -> int:
    return ((wf + 7) // 8) * ((hf + 3) // 4)


def workspace_for(tex: Texture, mode: int, filt: int, wf: int, hf: int, frames: int, device) -> torch.Tensor | None:
    """Device scratch for ctf_params.workspace_dev (the work lists of the lean COLLAB / Mask
    bilinear kernels), or None where the path does not use one."""
    if mode not in (MODE_COLLAB, MODE_BOX, MODE_MASK16, MODE_MASK11) or filt != FILTER_BILINEAR:
        return None
    nbytes = load_library().ctf_filter_workspace_bytes(wf, hf, frames)
    return torch.empty(nbytes, device=device, dtype=torch.uint8)


def _set_workspace(p: ctf_params, ws: torch.Tensor | None):
    if ws is not None:
        p.workspace_dev = ws.data_ptr()
        p.workspace_bytes = ws.numel() * ws.element_size()


def _call_workspace(tex, mode, filt, wf, hf, frames, device, workspace, stream):
    """The call's work-list scratch: a caller tensor, None, or (workspace=True) one allocated
    here.  A scratch allocated here is released when the call returns while the kernels still
    use it on `stream`; record_stream keeps the caching allocator from reusing the block until
    the work queued on that stream so far has finished."""
    if isinstance(workspace, torch.Tensor):
        return workspace
    if workspace is not True:
        return None
    ws = workspace_for(tex, mode, filt, wf, hf, frames, device)
    if ws is not None and stream is not None:
        ws.record_stream(stream)
    return ws


_U32_DTYPES = tuple(d for d in (torch.int32, getattr(torch, "uint32", None)) if d is not None)


def check_buffers(uv4: torch.Tensor, grad: torch.Tensor | None, out: torch.Tensor, rec: torch.Tensor | None,
                  debug: dict | None = None):
    """Validate the caller's buffers against the geometry uv4 = [F][Hf][Wf][2] before the C call.

    The C ABI takes plain pointers and sizes (include/ctf.h), so an undersized, mistyped or
    foreign-device buffer would be read or written out of bounds by the kernels instead of
    failing; this is where the binding turns that into a ValueError.  Pure host logic (no CUDA
    call): out / rec / debug buffers may be larger than needed (flat buffers are fine)."""
    if uv4.dim() != 4 or uv4.dtype != torch.float32 or uv4.shape[3] != 2:
        raise ValueError("uv must be float32 [F][Hf][Wf][2] (or [Hf][Wf][2])")
    frames, hf, wf = uv4.shape[0], uv4.shape[1], uv4.shape[2]
    if frames <= 0 or hf <= 0 or wf <= 0:
        raise ValueError("empty frame geometry")
    px = frames * hf * wf
    waves = frames * ((hf + 3) // 4) * ((wf + 7) // 8)
    need = [("grad", grad, (torch.float16,), 4 * px, True),
            ("out", out, (torch.float32,), 4 * px, False),
            ("rec", rec, _U32_DTYPES, waves, False)]
    for k, n in (("produced_id", px), ("selection", px), ("unread", 1)):
        if debug is not None and debug.get(k) is not None:
            need.append((k, debug[k], _U32_DTYPES, n, False))
    for name, t, dtypes, numel, exact in need:
        if t is None:
            continue
        if t.dtype not in dtypes:
            raise ValueError(f"{name} must be {' or '.join(str(d) for d in dtypes)}, got {t.dtype}")
        if (t.numel() != numel) if exact else (t.numel() < numel):
            raise ValueError(f"{name} holds {t.numel()} elements, the geometry needs {'' if exact else '>= '}{numel}")
        if t.device != uv4.device:
            raise ValueError(f"{name} is on {t.device}, uv on {uv4.device}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")


def filter_batch(tex: Texture, uv: torch.Tensor, grad: torch.Tensor | None, mode: int, fallback: int = FB_CPLUS,
                 flags: int = 0, seed: int = 0, frame_index: int = 0, out: torch.Tensor | None = None,
                 rec: torch.Tensor | None = None, debug: dict | None = None,
                 stream: torch.cuda.Stream | None = None, filter: int = FILTER_BILINEAR, max_evals: int = 1,
                 workspace: torch.Tensor | bool | None = True, row0: int = 0):
    """uv: float32 [F][Hf][Wf][2] (or [Hf][Wf][2]); grad: float16 [..][4] or None.
    row0: frame row of the buffers' first row (strip sharding; a multiple of 4).
    Returns (out float32 [..][4], rec int32 [F][nwy][nwx]).  `debug` may hold tensors
    'produced_id', 'selection' (int32, pixel-shaped) and 'unread' (int32 [1]).
    workspace: True = allocate the path's scratch (workspace_for) for this call, a tensor =
    use it, None / False = none (the record buffer doubles as the work list)."""
    lib = load_library()
    single = uv.dim() == 3
    uv4 = uv.unsqueeze(0) if single else uv
    if uv4.dim() != 4:
        raise ValueError("uv must be float32 [F][Hf][Wf][2] (or [Hf][Wf][2])")
    frames, hf, wf = uv4.shape[0], uv4.shape[1], uv4.shape[2]
    if out is None:
        out = torch.empty((frames, hf, wf, 4), device=uv.device, dtype=torch.float32)
    if rec is None:
        rec = torch.empty((frames, (hf + 3) // 4, (wf + 7) // 8), device=uv.device, dtype=torch.int32)
    check_buffers(uv4, grad, out, rec, debug)
    p = ctf_params(mode, fallback, flags, frame_index, seed, filter, max_evals)
    p.row0 = row0
    _set_workspace(p, _call_workspace(tex, mode, filter, wf, hf, frames, uv.device, workspace, stream))
    dbg = None
    if debug is not None:
        dbg = ctf_debug(_ptr(debug.get("produced_id")), _ptr(debug.get("selection")), _ptr(debug.get("unread")))
        p.flags |= FLAG_DEBUG
    rc = lib.ctf_filter_batch(ctypes.byref(tex.desc), _ptr(uv4), _ptr(grad), wf, hf, frames, ctypes.byref(p),
                              _ptr(out), _ptr(rec), ctypes.byref(dbg) if dbg is not None else None,
                              _stream(stream))
    _check("ctf_filter_batch", rc)
    if single:
        return out[0], rec[0]
    return out, rec


def filter_frame(tex: Texture, uv: torch.Tensor, grad: torch.Tensor | None, mode: int, fallback: int = FB_CPLUS,
                 flags: int = 0, seed: int = 0, frame_index: int = 0, out: torch.Tensor | None = None,
                 rec: torch.Tensor | None = None, debug: dict | None = None,
                 stream: torch.cuda.Stream | None = None, filter: int = FILTER_BILINEAR, max_evals: int = 1,
                 workspace: torch.Tensor | bool | None = True, row0: int = 0):
    """One frame through ctf_filter_frame.  uv float32 [Hf][Wf][2]; workspace and row0 as filter_batch."""
    lib = load_library()
    if uv.dim() != 3:
        raise ValueError("filter_frame: uv must be float32 [Hf][Wf][2]")
    hf, wf = uv.shape[0], uv.shape[1]
    if out is None:
        out = torch.empty((hf, wf, 4), device=uv.device, dtype=torch.float32)
    if rec is None:
        rec = torch.empty(((hf + 3) // 4, (wf + 7) // 8), device=uv.device, dtype=torch.int32)
    check_buffers(uv.unsqueeze(0), grad, out, rec, debug)
    p = ctf_params(mode, fallback, flags, frame_index, seed, filter, max_evals)
    p.row0 = row0
    _set_workspace(p, _call_workspace(tex, mode, filter, wf, hf, 1, uv.device, workspace, stream))
    dbg = None
    if debug is not None:
        dbg = ctf_debug(_ptr(debug.get("produced_id")), _ptr(debug.get("selection")), _ptr(debug.get("unread")))
        p.flags |= FLAG_DEBUG
    rc = lib.ctf_filter_frame(ctypes.byref(tex.desc), _ptr(uv), _ptr(grad), wf, hf, ctypes.byref(p), _ptr(out),
                              _ptr(rec), ctypes.byref(dbg) if dbg is not None else None, _stream(stream))
    _check("ctf_filter_frame", rc)
    return out, rec


def stats(rec: torch.Tensor, wf: int, hf: int, frames: int = 1, out: torch.Tensor | None = None,
          ref: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None) -> dict:
    """ctf_stats: totals of `frames` frames of records (+ error of out vs ref).  Synchronises."""
    lib = load_library()
    st = ctf_frame_stats()
    rc = lib.ctf_stats(_ptr(rec), wf, hf, frames, _ptr(out), _ptr(ref), ctypes.byref(st), _stream(stream))
    _check("ctf_stats", rc)
    return st.to_dict()


class HostPipeline:
    """ctf_filter_frames_host: host buffers in, host buffers out (copies inside the call)."""

    def __init__(self, wf: int, hf: int, chunk_frames: int, with_grad: bool, device="cuda"):
        lib = load_library()
        self.wf, self.hf, self.chunk = wf, hf, chunk_frames
        nbytes = lib.ctf_host_workspace_bytes(wf, hf, chunk_frames, int(with_grad))
        if nbytes == 0:
            raise ValueError("bad pipeline geometry")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)

    def run(self, tex: Texture, uv_host: torch.Tensor, grad_host: torch.Tensor | None, out_host: torch.Tensor,
            rec_host: torch.Tensor | None, mode: int, fallback: int = FB_CPLUS, flags: int = 0, seed: int = 0,
            frame_index: int = 0, stream: torch.cuda.Stream | None = None, filter: int = FILTER_BILINEAR,
            max_evals: int = 1, row0: int = 0):
        lib = load_library()
        for t in (uv_host, grad_host, out_host, rec_host):
            if t is not None and (t.is_cuda or not t.is_contiguous()):
                raise ValueError("host pipeline expects contiguous CPU (ideally pinned) tensors")
        if uv_host.dim() != 4 or tuple(uv_host.shape[1:3]) != (self.hf, self.wf):
            raise ValueError(f"uv_host must be [F][{self.hf}][{self.wf}][2] (the pipeline's geometry)")
        check_buffers(uv_host, grad_host, out_host, rec_host)   # rec_host may be None (records not copied back)
        frames = uv_host.shape[0]
        p = ctf_params(mode, fallback, flags, frame_index, seed, filter, max_evals)
        p.row0 = row0
        hp = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        rc = lib.ctf_filter_frames_host(ctypes.byref(tex.desc), hp(uv_host), hp(grad_host), self.wf, self.hf,
                                        frames, self.chunk, ctypes.byref(p), hp(out_host), hp(rec_host),
                                        ctypes.c_void_p(self.workspace.data_ptr()), self.workspace.numel(),
                                        _stream(stream))
        _check("ctf_filter_frames_host", rc)
