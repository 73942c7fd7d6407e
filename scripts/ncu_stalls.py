#!/usr/bin/env python
"""Top source lines of one ncu report by a stall reason.  usage: ncu_stalls.py <rep> [reason]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No" and "Instructions Executed" in r)
h = rows[hi]
iS, iR = h.index("Warp Stall Sampling (All Samples)"), h.index(reason)


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


out = [(num(r[iR]), num(r[iS]), r[0], r[1].strip()[:110]) for r in rows[hi + 1:] if r and r[0].isdigit()]
tot = sum(x[1] for x in out)
for x in sorted(out, reverse=True)[:12]:
    print(f"{reason} {100 * x[0] / tot:5.1f}%  all {100 * x[1] / tot:5.1f}%  L{x[2]} {x[3]}")
