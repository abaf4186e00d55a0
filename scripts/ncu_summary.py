"""Summarise an ncu --set full report: key metrics + per-wave instruction profile.

usage: python scripts/ncu_summary.py gpurun_out/prof_TAG.ncu-rep [waves_in_launch] [--sass out.txt]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "launch__grid_size", "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in KEYS or h == "Kernel Name":
                d[h] = (vals[i], units[i])
        res.append(d)
    return res


def sass_profile(rep, waves, out_path=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, ist = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    tot = 0
    lines = []
    for r in rows[2:]:
        if len(r) <= ia:
            continue
        try:
            n = int(r[ia])
        except ValueError:
            continue
        tot += n
        lines.append((n / waves, int(r[ist] or 0), r[isrc]))
    if out_path:
        with open(out_path, "w") as f:
            for n, st, src in lines:
                f.write(f"{n:8.3f} {st:7d}  {src}\n")
    return tot


if __name__ == "__main__":
    rep = sys.argv[1]
    waves = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for d in raw(rep):
        for k in ["Kernel Name"] + KEYS:
            if k in d:
                print(f"{k:90s} {d[k][0]} {d[k][1]}")
    if waves:
        sp = sys.argv[sys.argv.index("--sass") + 1] if "--sass" in sys.argv else None
        tot = sass_profile(rep, waves, sp)
        print(json.dumps({"warp_instructions": tot, "per_wave": tot / waves}))
