#!/usr/bin/env python3
"""Stall-reason breakdown of an ncu source page (SASS), by code region."""
import csv, re, collections, subprocess, sys
rep = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
isrc = hdr.index('Source'); iss = hdr.index('Warp Stall Sampling (All Samples)'); iex = hdr.index('Instructions Executed')
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
ri = [hdr.index(h) for h in reasons]
f = lambda v: float(v) if v not in ('', None) else 0.0
tot = sum(f(r[iss]) for r in data)
tot_r = collections.Counter()
for r in data:
    for h, i in zip(reasons, ri): tot_r[h] += f(r[i])
print("overall:", {k[6:]: round(v / tot * 100, 1) for k, v in tot_r.most_common(8)})
for w0 in range(0, len(data), W):
    blk = data[w0:w0 + W]
    s = sum(f(r[iss]) for r in blk)
    if s / tot < 0.015: continue
    ops = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', r[isrc].strip()).split(' ')[0].split('.')[0] for r in blk)
    rs = collections.Counter()
    for r in blk:
        for h, i in zip(reasons, ri): rs[h[6:]] += f(r[i])
    print(f"{w0:5d} {s/tot*100:5.1f}% {dict(ops.most_common(4))} | " +
          " ".join(f"{k}:{v/s*100:.0f}" for k, v in rs.most_common(4)))
