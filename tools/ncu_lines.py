"""Per-source-line stall summary of an ncu report (--page source --csv --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = {}
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if len(r) < 5 or r[0] == "" or hdr is None:
        continue
    try:
        n = int(r[4] or 0)
    except ValueError:
        continue
    d = agg.setdefault((fname, r[0], r[1][:70]), {"_n": 0})
    d["_n"] += n
    for i, x in enumerate(hdr):
        if x.startswith("stall_") and "Not Issued" not in x:
            try:
                d[x] = d.get(x, 0) + int(r[i] or 0)
            except ValueError:
                pass
tot = sum(d["_n"] for d in agg.values()) or 1
allr = {}
for d in agg.values():
    for x, v in d.items():
        if x != "_n":
            allr[x] = allr.get(x, 0) + v
print("samples", tot, sorted(((round(100 * v / tot, 1), x[6:]) for x, v in allr.items()), reverse=True)[:8])
for k, d in sorted(agg.items(), key=lambda t: -t[1]["_n"])[:top]:
    ts = sorted(((v, x) for x, v in d.items() if x != "_n"), reverse=True)[:3]
    print(f"{d['_n']:7d} {100 * d['_n'] / tot:5.1f}% {k[0]}:{k[1]:>4} {k[2][:60]:60s}", [(x[6:], v) for v, x in ts])
