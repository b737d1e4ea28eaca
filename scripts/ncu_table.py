#!/usr/bin/env python3
"""One markdown row per profiled launch of ncu --set full reports: duration, issue-slot and
pipe utilisation (FP32 FMA / FP64 / ALU), DRAM traffic and bandwidth, occupancy, registers.

usage: ncu_table.py report.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FP32 fma pipe %", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %", 1),
    ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    data = list(csv.reader(io.StringIO(txt)))
    if len(data) < 3:
        return []
    h = data[0]
    units = data[1]
    out = []
    for r in data[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "").split("::")[-1]
        vals = []
        for key, _, scale in COLS:
            if key not in h:
                vals.append(None)
                continue
            raw = r[h.index(key)].replace(",", "")
            u = units[h.index(key)]
            try:
                v = float(raw)
            except ValueError:
                vals.append(None)
                continue
            if key.startswith("dram__bytes"):  # normalise to bytes
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
            if key == "gpu__time_duration.sum":
                v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
            vals.append(v * scale)
        out.append((name, vals))
    return out


def main(reps):
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM GB/s |")
    print("|---" * (len(COLS) + 2) + "|")
    for rep in reps:
        for name, v in rows(rep):
            gbs = ""
            if v[0] and v[5] is not None and v[6] is not None:
                gbs = f"{(v[5] + v[6]) * 1e6 / (v[0] * 1e-6) / 1e9:.0f}"
            cells = [f"{x:.1f}" if isinstance(x, float) else "-" for x in v]
            print(f"| `{name}` | " + " | ".join(cells) + f" | {gbs} |")


if __name__ == "__main__":
    main(sys.argv[1:])
