"""Static per-kernel summary of libctf.so (no GPU needed): ptxas registers / spills / shared
memory from build_ptxas.log, and the SASS opcode mix from `cuobjdump -sass`.

    python scripts/sass_static.py [--all] > profiles/<round>/sass_static.txt

By default only the kernels the release BC1 / latent-MLP bilinear COLLAB paths launch (DBG =
false) and the bicubic kernels are listed; --all lists every instantiation.  Static counts are
instructions in the binary, not executed instructions (ncu's `inst_executed` is that)."""
from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2506_17770_b200" / "libctf.so"
LOG = ROOT / "paper_2506_17770_b200" / "build_ptxas.log"
FAMILIES = [
    ("tcgen05/UTC", r"^UTC"), ("HMMA", r"^HMMA"), ("LDSM", r"^LDSM"), ("FFMA2/FADD2/FMUL2", r"^F(FMA|ADD|MUL)2"),
    ("FFMA/FADD/FMUL", r"^F(FMA|ADD|MUL)$"), ("LDG", r"^LDG"), ("STG", r"^STG"), ("LDS", r"^LDS$"),
    ("STS", r"^STS"), ("ATOMS", r"^ATOMS"), ("ATOMG/RED", r"^(ATOMG|RED)"), ("SHFL", r"^SHFL"),
    ("VOTE", r"^VOTE"), ("REDUX", r"^REDUX"), ("POPC", r"^POPC"), ("PRMT", r"^PRMT"), ("BRA", r"^BRA"),
    ("LDL/STL", r"^(LDL|STL)"), ("UBLKCP/UTMA", r"^(UBLKCP|UTMA)"), ("MUFU", r"^MUFU"),
]


def demangle(names):
    try:
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
        return r.stdout.splitlines()
    except Exception:
        return list(names)


def ptxas_info():
    """mangled name -> (registers, spill stores, spill loads, smem bytes) from build_ptxas.log."""
    info, cur, spill = {}, None, (0, 0)
    for line in LOG.read_text().splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur, spill = m.group(1), (0, 0)
            continue
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1) if cur is None or m.group(1) == cur else cur
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spill = (max(spill[0], int(m.group(1))), max(spill[1], int(m.group(2))))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            sm = re.search(r"(\d+) bytes smem", line)
            info[cur] = (int(m.group(1)), spill[0], spill[1], int(sm.group(1)) if sm else 0)
            cur = None
    return info


def sass_mix():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    mix, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            mix[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m and cur:
            mix[cur][m.group(2)] += 1
    return mix


def main():
    everything = "--all" in sys.argv
    info, mix = ptxas_info(), sass_mix()
    names = sorted(mix)
    pretty = dict(zip(names, demangle(names)))
    print("# static SASS / ptxas summary of libctf.so (sm_100a); instructions in the binary, not executed")
    print("# regs / spill st / spill ld / static smem from build_ptxas.log (the kernel's own frame; out-of-line callees not included)")
    for n in names:
        p = pretty[n]
        targs = p.split("(")[0].split("<", 1)[-1]
        if not everything and (("collab_" in p and targs.startswith("true")) or "stats" in p):
            continue   # DBG instantiations (first template argument true) and the stats kernels
        c = mix[n]
        total = sum(c.values())
        r = info.get(n)
        head = f"regs {r[0]:3d}  spill st/ld {r[1]:3d}/{r[2]:3d} B  smem {r[3]:6d} B" if r else "regs ?"
        fams = []
        for label, rx in FAMILIES:
            k = sum(v for op, v in c.items() if re.match(rx, op))
            if k:
                fams.append(f"{label} {k}")
        print(f"\n{p}\n    {head}  SASS {total}\n    " + ", ".join(fams))


if __name__ == "__main__":
    main()
