"""Per-CUDA-source-line executed warp instructions (per wave) from an ncu report.

usage: python scripts/ncu_lines.py REPORT WAVES [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, waves = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
import os
kf = ["-k", os.environ["NCU_KERNEL"]] if os.environ.get("NCU_KERNEL") else []
if os.environ.get("NCU_SKIP"):
    kf += ["--launch-skip", os.environ["NCU_SKIP"], "--launch-count", "1"]
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = None
agg = defaultdict(float)
src_text = {}
hdr = None
cur_line = None
seen = set()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # rows with a line number carry the CUDA line; SASS rows follow with empty line number
    if r[0]:
        cur_line = (cur_file, int(r[0]))
        src_text[cur_line] = r[1]
    try:
        n = float(r[7]) if r[7] else 0.0
    except ValueError:
        n = 0.0
    if r[2] and cur_line and r[2] not in seen:
        seen.add(r[2])
        agg[cur_line] += n
tot = sum(agg.values())
print(f"total per wave: {tot / waves:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / waves:7.2f}  {k[0]}:{k[1]:<5d} {src_text.get(k, '')[:110]}")
