"""Per-kernel DRAM traffic from an ncu CSV of dram__bytes_read.sum, dram__bytes_write.sum and
gpu__time_duration.sum (one row per metric and launch): totals, per launch, GB/s.
usage: python tools/ncu_traffic.py dram.csv [kernel-substring]"""
import collections
import csv
import json
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
want = sys.argv[2] if len(sys.argv) > 2 else ""
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}
per = collections.defaultdict(dict)
names = {}
for r in csv.DictReader(rows):
    if want not in r["Kernel Name"]:
        continue
    key = r["ID"]
    names[key] = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r.get("Metric Unit", ""), 1.0)
    per[key][r["Metric Name"]] = v
rd = sum(p.get("dram__bytes_read.sum", 0.0) for p in per.values())
wr = sum(p.get("dram__bytes_write.sum", 0.0) for p in per.values())
tm = sum(p.get("gpu__time_duration.sum", 0.0) for p in per.values())
n = len(per)
out = {"launches": n, "dram_read_gb": rd / 1e9, "dram_write_gb": wr / 1e9, "gb_per_launch": (rd + wr) / 1e9 / max(1, n),
       "device_s": tm, "dram_gbs": (rd + wr) / max(tm, 1e-30) / 1e9}
print(json.dumps(out, indent=1))
