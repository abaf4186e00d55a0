"""Per-kernel share of an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[hdr.index("Kernel Name")].split("(")[0]
        tot[k] += float(r[hdr.index("Metric Value")].replace(",", ""))
        cnt[k] += 1
s = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k] / s * 100:6.1f} %  {cnt[k]:4d} launches  {tot[k] / cnt[k] / 1e3:9.1f} us/launch  {k}")
