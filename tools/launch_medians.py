"""Median duration per kernel from an ncu --metrics gpu__time_duration.sum --csv launch list:
python tools/launch_medians.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x["Metric Name"] == "gpu__time_duration.sum":
            d[x["Kernel Name"].split("(")[0][:60]].append(float(x["Metric Value"]) / 1e3)
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    v = sorted(v)
    print(f"{len(v):4d}  median {v[len(v) // 2]:8.2f} us  {k}")
