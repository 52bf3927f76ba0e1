"""Render tools/bench_resample.py's JSON lines as the config-5 table of profiles/ (GB/s | ms per cell).

    python tools/resample_table.py profiles/r1_resample_microbench.jsonl > profiles/r1_resample_microbench.txt
"""
import collections
import json
import sys

SCHEMES = ["systematic", "stratified", "multinomial", "residual", "residual_stratified", "residual_systematic"]
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
import json as _json, os as _os
peak = _json.load(open(_os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
print("# Config 5: resample + in-place copy via smc_resample (counts + parents + 32-byte row copy fused into pass C),")
print("# 1 B200, CUDA events, mean of 20 calls (5 at 2^26+); cell = GB/s | ms, GB/s = algorithmic bytes (N*(8 W +")
print(f"# 4 counts + 4 parents) + 64 per moved row) / time; HBM peak {peak} GB/s (MEASURED_PEAKS.json).")
print(f"# Raw lines: {sys.argv[1].split('/')[-1]} (tools/bench_resample.py)")
by = collections.defaultdict(dict)
for d in rows:
    by[d["weights"]][(d["log2n"], d["scheme"])] = d
for kind in ["uniform", "skewed1", "skewed3", "degenerate"]:
    if kind not in by:
        continue
    print(f"\n## weights: {kind}")
    print("log2N " + "".join(f"{s:>22s}" for s in SCHEMES))
    for lg in sorted({k[0] for k in by[kind]}):
        cells = []
        for s in SCHEMES:
            d = by[kind].get((lg, s))
            cells.append(f"{d['GBps']:>10.0f} | {d['ms']:>9.3f}" if d else " " * 22)
        print(f"{lg:>5d} " + "".join(cells))
