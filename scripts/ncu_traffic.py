"""Write profiles/ncu_traffic.json (the bench's `roofline.traffic`) from an ncu --set full report.

usage: python scripts/ncu_traffic.py gpurun_out/prof_TAG.ncu-rep [frames width height]

The report must hold the kernels of ONE ctf_filter_batch call (scripts/gpu_bench.sh captures
`-k regex:ctf_collab_ -s 3 -c 3`: the lean exact kernel and the two rest passes).
DRAM bytes are summed over those launches; bench.py reads the total as the per-call traffic.
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
from ncu_summary import raw  # noqa: E402


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1}


def scaled(v):
    """(value string, unit) from ncu_summary.raw -> bytes or seconds."""
    return float(v[0].replace(",", "")) * SCALE[v[1]]


def main():
    rep = sys.argv[1]
    frames, wf, hf = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (64, 3840, 2160)
    rows = raw(rep)
    per = {}
    inst = {}
    rd = wr = ms = 0.0
    for r in rows:
        name = r["Kernel Name"][0].split("(")[0].strip()
        b_r, b_w = scaled(r["dram__bytes_read.sum"]), scaled(r["dram__bytes_write.sum"])
        prev = per.get(name, [0.0, 0.0])
        per[name] = [prev[0] + b_r, prev[1] + b_w]   # the frame groups' launches of one kernel summed
        k_inst = float(r["smsp__inst_executed.sum"][0].replace(",", ""))
        inst[name] = inst.get(name, 0.0) + k_inst
        rd += b_r
        wr += b_w
        ms += scaled(r["gpu__time_duration.sum"]) * 1e3
    waves = frames * ((wf + 7) // 8) * ((hf + 3) // 4)
    alg = frames * wf * hf * 32 + waves * 4
    out = {
        "source": f"ncu --set full, {rep}: the kernels of one {frames}-frame bench step, DRAM bytes summed",
        "frames": frames, "width": wf, "height": hf, "per_kernel": per,
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": alg, "duration_ms_under_ncu": ms,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "warp_inst_per_kernel": inst, "warp_inst_per_launch": sum(inst.values()),
        "warp_inst_per_wave": sum(inst.values()) / waves,
    }
    p = pathlib.Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
