"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    agg.setdefault(r[ki].split("(")[0].replace("<unnamed>::", ""), []).append(float(r[vi].replace(",", "")))
tot = 0.0
for k, v in agg.items():
    print(f"{k[:60]:60s} n={len(v):3d} mean_us={sum(v) / len(v) / 1e3:9.1f} last_us={v[-1] / 1e3:9.1f}")
