"""Summarise an ncu --metrics gpu__time_duration.sum launch list (per-kernel mean us)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
im = hdr.index("Metric Name") if "Metric Name" in hdr else None
d = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > iv and (im is None or r[im] == "gpu__time_duration.sum"):
        d[r[ik].split("(")[0][:70]].append(float(r[iv].replace(",", "")) / 1e3)
tot = 0
for k, v in d.items():
    m = sum(v) / len(v); tot += m
    print(f"{len(v):4d} {m:9.2f} us  {k}")
print(f"sum of means {tot:.2f} us")
