"""ncu captures that bench.py folds into its line (profiles/move_ncu.json, profiles/gmm_mh_ncu.json).

Each JSON carries the library's source hash (paper_1306_5583_b200._build.source_hash) at capture
time; bench.py uses a capture only while the kernel sources still hash the same, so a kernel change
never reuses a stale profile silently.

    python tools/capture_profiles.py --commit <sha>        (on the GPU box; needs ncu)
"""

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NCU = "/usr/local/cuda/bin/ncu"


def ncu_metrics(kernel_regex, metrics, cmd, skip=0):
    out = subprocess.run([NCU, "--metrics", ",".join(metrics), "--clock-control", "none", "-k", f"regex:{kernel_regex}",
                          "-s", str(skip), "-c", "1", "--csv", *cmd], capture_output=True, text=True, cwd=ROOT)
    text = out.stdout[out.stdout.find('"ID"'):]
    vals = {}
    for r in csv.DictReader(io.StringIO(text)):
        vals[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        vals["_kernel"] = r["Kernel Name"]
    if not vals:
        raise RuntimeError(f"ncu produced no metrics:\n{out.stdout[-2000:]}\n{out.stderr[-2000:]}")
    return vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--commit", default="unknown")
    args = ap.parse_args()
    from paper_1306_5583_b200 import _build
    h = _build.source_hash()
    n = 1 << 24
    m = ncu_metrics("k_pf_move", ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                                  "gpu__time_duration.sum"],
                    [sys.executable, "tools/prof_step.py", str(n), "6"], skip=4)
    move = {"kernel": m["_kernel"], "n": n, "dram_bytes_read": m["dram__bytes_read.sum"],
            "dram_bytes_write": m["dram__bytes_write.sum"], "warp_inst": m["smsp__inst_executed.sum"],
            "inst_per_particle": m["smsp__inst_executed.sum"] * 32 / n,
            "duration_us_under_ncu": m["gpu__time_duration.sum"] / 1e3, "source_hash": h, "commit": args.commit,
            "source": "ncu --metrics ... --clock-control none -k regex:k_pf_move -s 4 -c 1 python tools/prof_step.py "
                      f"{n} 6 (the 5th move: after a resample, the uniform-count kernel)"}
    with open(os.path.join(ROOT, "profiles", "move_ncu.json"), "w") as f:
        json.dump(move, f, indent=1)
    ng, nd = 1 << 20, 1000
    g = ncu_metrics("k_gmm_mh", ["sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                                 "smsp__inst_executed.sum", "gpu__time_duration.sum"],
                    [sys.executable, "tools/bench_gmm.py", "--T", "3", "--seeds", "0"], skip=3)
    gmm = {"kernel": g["_kernel"], "n": ng, "nd": nd, "r": 4,
           "fp64_thread_inst": g["sm__inst_executed_pipe_fp64.sum"] * 32,
           "fp64_pipe_pct": g["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
           "warp_inst": g["smsp__inst_executed.sum"], "duration_us_under_ncu": g["gpu__time_duration.sum"] / 1e3,
           "source_hash": h, "commit": args.commit,
           "source": "ncu --metrics ... -k regex:k_gmm_mh -s 3 -c 1 python tools/bench_gmm.py --T 3 --seeds 0 "
                     "(the first MH block of iteration 2 at N=2^20, 1000 points, 4 components)"}
    with open(os.path.join(ROOT, "profiles", "gmm_mh_ncu.json"), "w") as f:
        json.dump(gmm, f, indent=1)
    print(json.dumps({"move": move, "gmm": gmm}))


if __name__ == "__main__":
    main()
