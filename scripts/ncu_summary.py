#!/usr/bin/env python3
"""Key metrics of an ncu --set full report (ncu -i REP --page details --csv), one block per launch.

usage: ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "No Eligible",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size",
        "Block Size", "Waves Per SM"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ii, mn, mv, mu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    cur = None
    for r in rows[1:]:
        if r[ii] != cur:
            cur = r[ii]
            print(f"\n### launch {cur}: `{r[ki].split('(')[0]}`\n")
            print("| metric | value |\n|---|---|")
        if r[mn] in WANT:
            print(f"| {r[mn]} | {r[mv]} {r[mu]} |")


if __name__ == "__main__":
    main(sys.argv[1])
