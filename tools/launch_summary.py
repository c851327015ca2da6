#!/usr/bin/env python3
"""Per-kernel launch counts, mean duration and share of the summed time from an
`ncu --metrics gpu__time_duration.sum --csv` launch list (cold-cache, serialised
launches: compare shares, not absolute times).  Usage: launch_summary.py CSV [TITLE]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iunit = hdr.index("Metric Unit")
tot, per = 0.0, {}
for r in rows[1:]:
    if r[imet] != "gpu__time_duration.sum":
        continue
    name = r[iname].split("(")[0].replace("rsr::", "")
    v = float(r[ival].replace(",", ""))
    unit_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[iunit]]
    per.setdefault(name, []).append(v * unit_us)
    tot += v * unit_us
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print("# per-launch times are cold-cache and serialised: compare shares")
for name, vs in per.items():
    print(f"{name:40s} launches={len(vs):3d} mean_us={sum(vs) / len(vs):9.1f} share={sum(vs) / tot:.3f}")
