#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

usage: summarize_launches.py launches.csv [> summary.md]
Times are ncu's serialised, cold-cache per-launch durations: use the SHARE of each kernel,
not the absolute sum, when comparing with bench.py's CUDA-event timings.
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        try:
            v = float(r[mi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("tjx::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {v[0]} | {v[1] / 1e6:.2f} | {100 * v[1] / tot:.1f}% |")
    print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e6:.2f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
