"""Summarise an ncu --csv launch list: the LAST occurrence of each step's kernels."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(per)
last = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sel = ids[-last:]
tot = sum(per[i]["gpu__time_duration.sum"] for i in sel)
for i in sel:
    d = per[i]
    t = d["gpu__time_duration.sum"]
    rb, wb = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
    print(f"{d['name'][:48]:48s} {t / 1e3:9.1f} us {100 * t / tot:5.1f}%  DRAM r {rb / 1e9:6.2f} GB w {wb / 1e9:6.2f} GB"
          f"  {(rb + wb) / t:7.0f} GB/s")
print(f"total {tot / 1e3:.1f} us")
