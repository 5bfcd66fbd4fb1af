#!/usr/bin/env python
"""Per-opcode instruction / stall-sample shares from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, rs = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rs.append(r)
ix = {h: j for j, h in enumerate(hdr)}
samp = lambda r: float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
inst = lambda r: float(r[ix["Instructions Executed"]] or 0)
tot = sum(samp(r) for r in rs)
ti = sum(inst(r) for r in rs)
by = collections.defaultdict(lambda: [0, 0])
for r in rs:
    op = [o for o in r[ix["Source"]].split() if not o.startswith("@")]
    op = op[0] if op else "?"
    by[op][0] += samp(r)
    by[op][1] += inst(r)
print("instructions", ti)
for op, (s, i) in sorted(by.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{op:22s} inst {100 * i / ti:5.1f}%  stall-samples {100 * s / tot:5.1f}%")
print("--- hottest instructions")
for r in sorted(rs, key=lambda r: -samp(r))[:12]:
    print(f"{100 * samp(r) / tot:5.1f}% exec={inst(r):>10.0f} {r[ix['Source']][:80]}")
