"""Per-kernel HBM roofline of one PF step at N = 2^24 (systematic): algorithmic bytes
over the kernel's time in the bench chain (launch list, last launch) and under ncu (cold, serialized),
with the ncu-measured DRAM traffic beside it.

    python tools/roofline_table.py profiles/r1_launches_pf_2e24.txt profiles/r1_ncu_dram_traffic.txt
"""
import sys

N = 1 << 24
import json as _json, os as _os
PEAK = _json.load(open(_os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]  # GB/s
# algorithmic bytes per launch (DESIGN.md §6 table; the move after a resample: lw is not read)
ALG = {
    "k_pf_move": N * (32 + 32 + 4 + 8 + 8 + 8),
    "k_rs_tiles": N * (8 + 8),
    "k_rs_counts": N * (8 + 4),
    "k_rs_ranks": N * (4 + 3),
    "k_rs_assign": N * (4 + 4),
    "k_rs_scan": 8192 * 16 * 2,
    "k_rs_zsp_scan": 8192 * 8 * 2,
    "k_lse_reduce": (N // 1024) * 24 + 148 * 24,
}


def key(name):
    for k in ALG:
        if k in name:
            return k
    return None


chain = {}
for line in open(sys.argv[1]):
    k = key(line.split(" n=")[0])
    if k and k not in chain:
        chain[k] = float(line.split("last_us=")[1])
ncu = {}
for line in open(sys.argv[2]):
    if line.startswith("#"):
        continue
    parts = line.split()
    k = key(parts[0] if parts[0] != "void" else parts[1])
    if k:
        ncu[k] = (float(parts[-3]), float(parts[-2]), float(parts[-1]))
print(f"# per-kernel HBM roofline, one PF step at N = 2^24 (systematic, resampled every step); peak {PEAK} GB/s")
print("# alg = algorithmic bytes per launch (DESIGN.md §6); chain = time in the bench's PF step (launch list, last")
print("# launch); ncu = cold serialized time and DRAM bytes from the ncu --set full capture")
print(f"{'kernel':16s} {'alg MB':>8s} {'chain us':>9s} {'GB/s':>7s} {'frac':>6s} {'ncu us':>8s} {'DRAM MB':>8s} {'DRAM GB/s':>9s}")
for k, b in ALG.items():
    t = chain.get(k)
    r, w, d = ncu.get(k, (0.0, 0.0, 0.0))
    gbs = b / (t * 1e-6) / 1e9 if t else 0.0
    print(f"{k:16s} {b / 1e6:8.1f} {t or 0:9.1f} {gbs:7.0f} {gbs / PEAK:6.2f} {d:8.1f} {r + w:8.1f} "
          f"{(r + w) * 1e6 / (d * 1e-6) / 1e9 if d else 0:9.0f}")
