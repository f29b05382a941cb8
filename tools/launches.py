"""Summarise an ncu --csv launch list: per-kernel time, DRAM bytes, achieved GB/s."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
k = OrderedDict()
for r in data:
    k.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = 0.0
for (i, name), m in k.items():
    if i < skip:
        continue
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    by = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot += t
    print(f"{i:3d} {t:9.1f} us {by/1e9:7.3f} GB {by/max(t,1e-9)/1e3:8.1f} GB/s  {name[:90]}")
print(f"total {tot:.1f} us")
