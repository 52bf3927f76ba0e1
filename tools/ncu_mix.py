"""Dynamic instruction mix of one kernel in an ncu report (from the source page's
per-SASS-line 'Instructions Executed'): python tools/ncu_mix.py rep.ncu-rep regex [per]."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0  # divide by (e.g.) warps of particles
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Address" in r and "Source" in r)
ai, si, ei = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
seen, mix = set(), collections.Counter()
for r in rows[rows.index(h) + 1:]:
    if len(r) > max(ai, si, ei) and r[ai].startswith("0x") and r[ai] not in seen:
        seen.add(r[ai])
        src = r[si].strip()
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        op = op.split(".")[0]
        mix[op] += int(r[ei]) if r[ei].isdigit() else 0
tot = sum(mix.values())
print(f"{kern}: {tot} warp-instructions ({tot / per:.1f} per unit)")
for op, c in mix.most_common(30):
    print(f"  {op:10s} {c:12d} {100.0 * c / tot:5.1f}%  {c / per:8.1f}/unit")
