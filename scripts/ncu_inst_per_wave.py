"""Reads an ncu --csv metrics dump on stdin; prints per-kernel warp-instructions per wave
(waves = F x 540 x 480, the 4K camera-path batch of scripts/time_libs.py)."""
import csv, sys
lib, F = sys.argv[1], int(sys.argv[2])
waves = F * 540 * 480  # (4K frames)
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = {}
for r in rows[1:]:
    k = r[ki].split("(")[0][:60]
    agg.setdefault((r[0], k), {})[r[mi]] = float(r[vi].replace(",", ""))
for (i, k), m in agg.items():
    print(f"{lib}: {k:60s} inst/wave {m.get('smsp__inst_executed.sum', 0) / waves:8.2f}  "
          f"us {m.get('gpu__time_duration.sum', 0) / 1e3:8.1f}  issue {m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}%")
