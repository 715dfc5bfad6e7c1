"""Per-config DRAM traffic and fma-heavy pipe use of ONE step from ncu launch lists.

    python tools/traffic_json.py profiles/r02_traffic.json CFG:launches.csv:K:UNITS ...

K = launches per step (the last K launches of the list are the last step),
UNITS = units of work per step.  Writes {CFG: {dram_bytes_per_unit,
step_time_us (cold-cache ncu replay), fmaheavy_time_weighted_pct, kernels: [...]}}.
bench.py reads dram_bytes_per_unit as roofline.traffic (x units per launch).
"""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0]})[r[mi]] = v
    return [per[i] for i in sorted(per)]


def main():
    out_path = sys.argv[1]
    try:
        out = json.load(open(out_path))
    except Exception:
        out = {}
    for spec in sys.argv[2:]:
        cfg, path, k, units = spec.split(":")
        ks = load(path)[-int(k):]
        t = sum(d["gpu__time_duration.sum"] for d in ks)
        rb = sum(d.get("dram__bytes_read.sum", 0) for d in ks)
        wb = sum(d.get("dram__bytes_write.sum", 0) for d in ks)
        fh = [d.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed") for d in ks]
        fmah = (sum(f * d["gpu__time_duration.sum"] for f, d in zip(fh, ks)) / t
                if all(f is not None for f in fh) else None)
        out[cfg] = {
            "dram_bytes_per_unit": (rb + wb) / int(units),
            "dram_read_bytes_per_step": rb, "dram_write_bytes_per_step": wb,
            "step_time_us": t / 1e3, "units_per_step": int(units),
            "fmaheavy_time_weighted_pct": fmah,
            "source": f"ncu launch list {path.split('/')[-1]} (last {k} launches = one step, "
                      "--clock-control none, cold-cache serialised replay)",
            "kernels": [{"name": d["name"], "us": d["gpu__time_duration.sum"] / 1e3,
                         "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                         "fmaheavy_pct": d.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed")}
                        for d in ks],
        }
        print(cfg, f"{(rb + wb) / int(units) / 1e6:.1f} MB/unit", f"{t / 1e3:.1f} us/step",
              f"fmaheavy {fmah:.1f}%" if fmah is not None else "")
    json.dump(out, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
