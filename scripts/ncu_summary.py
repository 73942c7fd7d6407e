#!/usr/bin/env python
"""Summarize an ncu report (full set) and an ncu launch-list CSV into markdown.

usage: scripts/ncu_summary.py <report.ncu-rep> [launches.csv] > profiles/<round>_<kernel>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Achieved Active Warps Per SM", "Grid Size", "Block Size", "SM Frequency",
        "DRAM Frequency", "Branch Efficiency", "Mem Busy", "Max Bandwidth"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    out = []
    det = list(csv.reader(io.StringIO(ncu([rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    kname = det[1][hdr.index("Kernel Name")] if len(det) > 1 else "?"
    out.append(f"## ncu --set full: `{kname[:120]}`\n")
    out.append("| metric | unit | value |\n|---|---|---|")
    seen = set()
    for row in det[1:]:
        if len(row) > 14 and row[12] in KEYS and row[12] not in seen:
            seen.add(row[12])
            out.append(f"| {row[12]} | {row[13]} | {row[14]} |")
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        h, units, vals = raw[0], raw[1], raw[2]
        out.append("")
        for k in RAW:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {units[i]} | {vals[i]} |")
    # source hot spots
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    try:
        sh = src[2]
        iS = sh.index("Warp Stall Sampling (All Samples)")
        iE = sh.index("Instructions Executed")
        st_cols = [i for i, x in enumerate(sh) if x.startswith("stall_") and "Not Issued" not in x]
        lines = []
        for r in src[3:]:
            if r and r[0]:
                try:
                    lines.append((int(r[0]), r[1].strip()[:80], int(r[iS]), int(r[iE]),
                                  {sh[i][6:]: int(r[i] or 0) for i in st_cols}))
                except ValueError:
                    pass
        tot = sum(x[2] for x in lines) or 1
        toti = sum(x[3] for x in lines) or 1
        out.append("\n### Source hot spots (stall samples, instructions)\n")
        out.append("| line | stall % | inst % | top stall reasons | source |\n|---|---|---|---|---|")
        for l in sorted(lines, key=lambda x: -x[2])[:15]:
            top = sorted(l[4].items(), key=lambda kv: -kv[1])[:3]
            out.append(f"| {l[0]} | {100 * l[2] / tot:.1f} | {100 * l[3] / toti:.1f} | "
                       f"{', '.join(f'{k} {100 * v / tot:.1f}' for k, v in top)} | `{l[1]}` |")
    except (IndexError, ValueError):
        pass
    if len(sys.argv) > 2:
        agg = defaultdict(list)
        with open(sys.argv[2]) as f:
            rows = [r for r in csv.reader(f) if len(r) > 10]
        h = rows[0]
        iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        for r in rows[1:]:
            if r[iM] == "gpu__time_duration.sum":
                name = r[iN].split("(")[0].replace("kvq::<unnamed>::", "")
                agg[name].append(float(r[iV].replace(",", "")))
        tot = sum(sum(v) for v in agg.values()) or 1
        out.append("\n### Launch list (ncu, cold-cache, serialized; compare shares)\n")
        out.append("| kernel | launches | mean ns | total share |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / tot:.1f}% |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
