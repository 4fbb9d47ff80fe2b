"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) by kernel:
launches, total ms, share.  usage: python tools/ncu_summary.py launches.csv [title]"""
import collections
import csv
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
agg = collections.OrderedDict()
n = 0
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    n += 1
    k = row["Kernel Name"].split("(")[0].replace("void ", "")
    if "spd::" not in k:
        k = k.split("<")[0]
    t = float(row["Metric Value"]) * (1e-3 if row.get("Metric Unit") == "ns" else 1.0)   # -> us
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"# {title}\n\nlaunches profiled: {n}; total device time {tot/1e3:.2f} ms (cold-cache, serialised)\n")
print("| kernel | launches | total ms | avg us | share |\n|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {v[0]} | {v[1]/1e3:.2f} | {v[1]/max(1,v[0]):.1f} | {100*v[1]/tot:.1f}% |")
