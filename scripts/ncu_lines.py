#!/usr/bin/env python3
"""Per-source-line instruction and stall shares of one kernel in an ncu report (-lineinfo build).

usage: ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
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
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        try:
            out.append((cur, int(r[0]), r[1][:90], int(r[7] or 0), int(r[4] or 0)))
        except ValueError:
            pass
    tot = sum(o[3] for o in out) or 1
    st = sum(o[4] for o in out) or 1
    print(f"total warp instructions {tot}, stall samples {st}")
    for o in sorted(out, key=lambda x: -x[3])[:top]:
        print(f"{o[0]}:{o[1]} inst {o[3] / tot * 100:.1f}% stall {o[4] / st * 100:.1f}%  {o[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
