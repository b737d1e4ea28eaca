#!/usr/bin/env python3
"""Per-source-line instructions and stall reasons (long/short scoreboard, wait, branch) of one
kernel in an ncu --set full report built with -lineinfo.

usage: ncu_stalls.py report.ncu-rep [top] [sort-column]
"""
import csv
import io
import subprocess
import sys

COLS = ["Instructions Executed", "Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_short_sb", "stall_wait",
        "stall_branch_resolving", "stall_mio", "stall_lg", "stall_math"]


def main(rep, top=40, key="Warp Stall Sampling (All Samples)"):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, idx, rows, src = None, None, {}, {}
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            idx = {c: r.index(c) for c in COLS if c in r}
            continue
        if idx is None or len(r) < 8 or not r[0]:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        vals = []
        for c in COLS:
            try:
                vals.append(float(r[idx[c]] or 0))
            except (KeyError, ValueError):
                vals.append(0.0)
        rows[(cur, ln)] = vals
        src[(cur, ln)] = r[1][:70]
    tot = [sum(v[i] for v in rows.values()) or 1 for i in range(len(COLS))]
    print("totals:", {c: int(t) for c, t in zip(COLS, tot)})
    k = COLS.index(key)
    print(f"{'line':28s} " + " ".join(f"{c[:10]:>10s}" for c in COLS))
    for (f, ln), v in sorted(rows.items(), key=lambda x: -x[1][k])[:top]:
        print(f"{f[:18]}:{ln:<5d}    " + " ".join(f"{100 * v[i] / tot[i]:10.2f}" for i in range(len(COLS))) + "  " + src[(f, ln)])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)")
