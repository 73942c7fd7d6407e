#!/usr/bin/env python
"""Per-source-line instruction counts and stall reasons of one ncu report (att_kernel).

usage: scripts/ncu_lines.py <report.ncu-rep> [units]   (units: tiles to normalise by)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No" and "Instructions Executed" in r)
h = rows[hi]
iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iW, iWI = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
st = [(i, x) for i, x in enumerate(h) if x.startswith("stall_")]
tot_st = defaultdict(float)
lines = []
for r in rows[hi + 1:]:
    if not r or not r[0].isdigit():
        continue
    def num(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    e = num(r[iE])
    sm = num(r[iS])
    for i, x in st:
        tot_st[x] += num(r[i])
    lines.append((int(r[0]), e, sm, r[1].strip()[:90], num(r[iW]), num(r[iWI])))
te = sum(x[1] for x in lines)
tw = sum(x[4] for x in lines)
print(f"shared wavefronts {tw:.0f} per unit {tw / units:.0f} (ideal {sum(x[5] for x in lines) / units:.0f})")
ts = sum(x[2] for x in lines)
print(f"warp instructions {te:.0f}  per unit {te / units:.0f}")
print("stall reasons (% of samples):")
for k, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:14]:
    print(f"  {k:40s} {100 * v / max(ts, 1):5.1f}")
print("top lines by instructions:")
for l in sorted(lines, key=lambda x: -x[1])[:40]:
    print(f"{l[0]:5d} inst {l[1] / units:6.0f}/u  wf {l[4] / units:5.0f}/u (ideal {l[5] / units:4.0f})  stall {100 * l[2] / max(ts, 1):5.1f}%  {l[3]}")
print("top lines by shared wavefronts:")
for l in sorted(lines, key=lambda x: -x[4])[:20]:
    print(f"{l[0]:5d} wf {l[4] / units:5.0f}/u (ideal {l[5] / units:4.0f})  {l[3]}")
print("top lines by stall samples:")
for l in sorted(lines, key=lambda x: -x[2])[:25]:
    print(f"{l[0]:5d} stall {100 * l[2] / max(ts, 1):5.1f}%  inst {l[1] / units:6.0f}/u  {l[3]}")
