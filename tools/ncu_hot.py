"""Top stalled SASS instructions of an ncu source-page CSV (--page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
data = []
for r in rows[2:]:
    try:
        n = int(r[iss] or 0)
    except ValueError:
        continue
    top = sorted(((int(r[h.index(x)] or 0), x[6:]) for x in reasons), reverse=True)[:3]
    data.append((n, r[ia][-5:], r[isrc][:70], top))
tot = sum(d[0] for d in data)
agg = {}
for r in rows[2:]:
    for x in reasons:
        try:
            agg[x] = agg.get(x, 0) + int(r[h.index(x)] or 0)
        except ValueError:
            pass
print("total samples", tot, {k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]})
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{d[0]:6d} {100 * d[0] / tot:5.1f}% {d[1]} {d[2]:70s} {d[3]}")
