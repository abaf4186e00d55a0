"""Build libctf.so (the CUDA hot path behind include/ctf.h) in-tree for sm_100a.

Translation units are compiled in parallel (the BC1 and latent-MLP kernel
instantiations are separate objects of ctf_filter.cu) and linked with a static
CUDA runtime, so the library loads without a GPU and without LD_LIBRARY_PATH.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libctf.so"
# (source, extra defines, object name)
UNITS = [
    ("ctf_abi.cu", [], "ctf_abi.o"),
    ("ctf_filter.cu", ["-DCTF_TU_FMT=1"], "ctf_filter_bc1.o"),
    ("ctf_filter.cu", ["-DCTF_TU_FMT=2"], "ctf_filter_mlp.o"),
    ("ctf_stats.cu", [], "ctf_stats.o"),
    ("ctf_bicubic.cu", ["-DCTF_TU_FMT=1"], "ctf_bicubic_bc1.o"),
    ("ctf_bicubic.cu", ["-DCTF_TU_FMT=2"], "ctf_bicubic_mlp.o"),
]
HEADERS = sorted(p.name for p in CSRC.iterdir() if p.suffix in (".cuh", ".h"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-v", "-I", str(ROOT / "include")]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / u[0] for u in UNITS] + [CSRC / h for h in HEADERS] + [ROOT / "include" / "ctf.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OBJ.mkdir(exist_ok=True)
    procs = []
    for src, defs, obj in UNITS:
        cmd = [NVCC, *ARCH, *CFLAGS, *defs, "-c", str(CSRC / src), "-o", str(OBJ / obj)]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    log = []
    failed = False
    for obj, p in procs:
        out, _ = p.communicate()
        log.append(f"==== {obj}\n{out}")
        failed |= p.returncode != 0
    (PKG / "build_ptxas.log").write_text("\n".join(log))
    if failed:
        sys.stderr.write("\n".join(log))
        raise RuntimeError("nvcc failed building libctf.so (see build_ptxas.log)")
    link = [NVCC, *ARCH, "-shared", "-cudart=static", "-o", str(LIB), *[str(OBJ / u[2]) for u in UNITS]]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link of libctf.so failed")
    if verbose:
        sys.stdout.write("\n".join(log))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
