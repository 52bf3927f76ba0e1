"""Top stall-sampled SASS lines of one kernel in an ncu report: python tools/ncu_hot.py rep.ncu-rep regex [n]."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Address" in r and "Source" in r)
ai, si = h.index("Address"), h.index("Source")
wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
seen, data = set(), []
for r in rows[rows.index(h) + 1:]:
    if len(r) > max(ai, si, wi, ei) and r[ai] not in seen and r[ai].startswith("0x"):
        seen.add(r[ai])
        data.append(r)
g = lambda r, i: int(r[i]) if r[i].isdigit() else 0
tot = sum(g(r, wi) for r in data)
print(f"{kern}: samples {tot}, warp-instr executed {sum(g(r, ei) for r in data)}")
for r in sorted(data, key=lambda r: -g(r, wi))[:top]:
    print(f"{g(r, wi):6d} {100.0 * g(r, wi) / max(tot, 1):5.1f}% {g(r, ei):9d}  {r[si][:90]}")
