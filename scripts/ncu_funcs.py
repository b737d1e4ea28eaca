#!/usr/bin/env python3
"""Per-function instruction / stall shares of one kernel in an ncu report (-lineinfo build):
source lines are attributed to the enclosing top-level function of their file.

usage: ncu_funcs.py report.ncu-rep [csrc dir]
"""
import csv
import io
import os
import re
import subprocess
import sys


def main(rep, csrc):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, out = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 9 or r[0] == "":
            continue
        try:
            out.append((cur, int(r[0]), int(r[7] or 0), int(r[4] or 0), int(r[8] or 0)))
        except ValueError:
            pass
    cache = {}

    def fn_of(f, line):
        path = os.path.join(csrc, f)
        if not os.path.exists(path):
            return f
        if f not in cache:
            cache[f] = open(path).read().split("\n")
        lines = cache[f]
        for i in range(min(line, len(lines)) - 1, -1, -1):
            s = lines[i]
            if s and not s[0].isspace() and "(" in s and not s.startswith(("//", "#", "}")):
                m = re.findall(r"(\w+)\(", s)
                if m:
                    return f"{f}:{m[0] if m[0] not in ('__launch_bounds__',) else m[-1]}"
        return f

    agg = {}
    for f, line, inst, stall, thr in out:
        a = agg.setdefault(fn_of(f, line), [0, 0, 0])
        a[0] += inst
        a[1] += stall
        a[2] += thr
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
        print(f"{k:48s} inst {100 * v[0] / ti:5.1f}%  stall {100 * v[1] / ts:5.1f}%  thread-inst {v[2] / 1e6:.0f}M")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "paper_2604_19982_b200/csrc")
