#!/bin/bash
# Stage-1 pair-class counts per k_screen launch (diagnostics build variants/stats, -DTJ_S1_STATS).
cp variants/stats/libtrijoin_b200.so paper_2604_19982_b200/
for c in B C D; do
  extra=""; [ "$c" = D ] && extra="--scale 0.05"
  python bench.py --config $c --no-cpu-baseline --no-e2e --steps 1 --warmup 0 $extra 2>&1 >/dev/null | grep S1STATS | tail -3
done
