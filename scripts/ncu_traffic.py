#!/usr/bin/env python3
"""DRAM traffic per launch of the kernels in ncu --set full reports -> profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic for the dominant kernel).

usage: ncu_traffic.py out.json report.ncu-rep [report.ncu-rep ...]
"""
import csv
import io
import json
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    for row in r[2:]:
        yield {k: (row[i], units[i]) for i, k in enumerate(h)}


def val(cell):
    v, u = cell
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


def main(out, reps):
    launches = []
    for rep in reps:
        for x in rows(rep):
            name = re.search(r"(k_\w+)", x["Kernel Name"][0])
            launches.append({
                "kernel": name.group(1) if name else x["Kernel Name"][0][:60],
                "report": rep.split("/")[-1],
                "dram_read_bytes": val(x["dram__bytes_read.sum"]),
                "dram_write_bytes": val(x["dram__bytes_write.sum"]),
                "duration_s": val(x["gpu__time_duration.sum"]),
            })
    for l in launches:
        l["dram_bytes"] = l["dram_read_bytes"] + l["dram_write_bytes"]
        l["dram_GBps"] = l["dram_bytes"] / l["duration_s"] / 1e9
    json.dump({"source": "ncu --set full --clock-control none (one launch per capture)", "launches": launches},
              open(out, "w"), indent=1)
    for l in launches:
        print(l["kernel"], l["report"], round(l["dram_bytes"] / 1e6, 1), "MB", round(l["dram_GBps"], 1), "GB/s")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
