"""Per-CUDA-source-line instruction counts of one kernel (ncu --print-source cuda,sass):
python tools/ncu_lines.py rep.ncu-rep regex [per] [top]."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res = "?", []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ei = r.index("Instructions Executed")
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and len(r) > ei and r[0] not in ("", "Function Name") and r[0].isdigit():
        n = int(r[ei]) if r[ei].isdigit() else 0
        smp = int(r[si]) if r[si].isdigit() else 0
        if n:
            res.append((n, smp, f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(x[0] for x in res)
stot = sum(x[1] for x in res)
print(f"{kern}: {tot / per:.1f} instr/unit over {len(res)} lines; samples {stot}")
for n, smp, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{n / per:8.1f} {100.0 * smp / max(stot, 1):5.1f}%  {loc:24s} {src}")
