"""CPU checks of the compiled kernels (ptxas report of the in-tree build, no GPU): the kernels
the BC1 bilinear COLLAB step launches keep the register budget their occupancy design assumes
(paired lean kernel 6 CTAs x 8 warps per SM -> <= 40 registers) without
spilling, and the hot kernels are built for sm_100a."""
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _ptxas():
    from paper_2506_17770_b200 import build
    build.build()
    info, cur, spill = {}, None, None
    for line in (ROOT / "paper_2506_17770_b200" / "build_ptxas.log").read_text().splitlines():
        m = re.search(r"Compiling entry function '(\S+)' for '(\w+)'", line)
        if m:
            cur, spill = (m.group(1), m.group(2)), None
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur and spill is None:
            spill = (int(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            info[cur[0]] = (cur[1], int(m.group(1)), spill or (0, 0))
            cur = None
    return info


def _demangled(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
    return dict(zip(r.stdout.splitlines(), names))


def test_hot_kernels_registers_and_spills():
    info = _ptxas()
    dm = _demangled(list(info))
    def get(prefix):
        hits = [k for k in dm if k.startswith(prefix)]
        assert len(hits) == 1, (prefix, hits)
        return info[dm[hits[0]]]
    # release, GRAD, not FORCE, BC1, List, not fused: the config-5 lean exact kernel
    arch, regs, (st, ld) = get("void ctf::ctf_collab_lean_kernel<false, true, false, 1, false, false>")
    assert arch == "sm_100a" and regs <= 40 and st == 0 and ld == 0, (arch, regs, st, ld)
    # the wide-window kernel (rest kernel, FALLBACK = true, BC1)
    arch, regs, (st, ld) = get("void ctf::ctf_collab_rest_kernel<false, true, 1>")
    assert arch == "sm_100a" and st == 0 and ld == 0, (arch, regs, st, ld)
    # every entry point is compiled for sm_100a only
    assert {v[0] for v in info.values()} == {"sm_100a"}
