"""Top SASS instructions of one kernel by warp-stall samples (ncu --set full report).

usage: python scripts/ncu_stalls.py REPORT regex:KERNEL
Columns: SASS index, share of all stall samples, instructions executed, SASS text."""
import csv, io, subprocess, sys
rep = sys.argv[1]; kern = sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; ist = hdr.index("Warp Stall Sampling (All Samples)"); isrc = hdr.index("Source"); ia = hdr.index("Instructions Executed")
data = []
seen_hdr = 0
for r in rows[2:]:
    if r and r[0] == "Kernel Name": break
    if len(r) <= ist: continue
    try: st = int(r[ist] or 0); n = int(r[ia] or 0)
    except ValueError: continue
    data.append((st, n, r[isrc].strip()))
tot = sum(d[0] for d in data)
print("total samples", tot)
for i, (st, n, src) in enumerate(data):
    pass
top = sorted(range(len(data)), key=lambda i: -data[i][0])[:40]
for i in sorted(top):
    st, n, src = data[i]
    print(f"{i:5d} {100*st/tot:5.1f}%  {n:>10d}  {src}")
