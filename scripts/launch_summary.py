#!/usr/bin/env python
"""Sum an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
    python scripts/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]][:70]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] += 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:8.3f} ms  x{cnt[k]:3d}  {k}")
print(f"total {sum(tot.values()):.3f} ms")
