"""Side-by-side min ms per (weights, log2 N, scheme) of tools/bench_resample.py runs of several
library variants: python tools/ab_resample_table.py prefix v1 v2 ... (files prefix_<v><rep>.jsonl)."""
import collections
import glob
import json
import sys

prefix, vs = sys.argv[1], sys.argv[2:]
d = collections.defaultdict(dict)
for v in vs:
    for f in glob.glob(f"{prefix}_{v}[0-9].jsonl"):
        for line in open(f):
            x = json.loads(line)
            k = (x["weights"], x["log2n"], x["scheme"])
            d[k].setdefault(v, []).append(x["ms"])
print(f"{'weights':10s} {'lg':>3s} {'scheme':20s} " + " ".join(f"{v:>8s}" for v in vs))
for k in sorted(d):
    print(f"{k[0]:10s} {k[1]:3d} {k[2]:20s} " + " ".join(f"{min(d[k].get(v, [0])):8.3f}" for v in vs))
