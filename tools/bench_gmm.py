"""Config 3: GMM SMC sampler, N = 2^20, 1000 synthetic points, T = 100, prior
annealing p = 2, Stratified at ESS/N < 0.5 (BASELINE.json configs[2]).

Reports wall time of initialize + 100 iterations (CUDA events, synced on both
sides), particle-iterations/s, the DS and PS log Z estimates, and the FP64
work: each MH block evaluates llh over n data x R components per particle, so
the likelihood evaluations per run = N * (1 + T * (1 + 3)) * n (init, reweight
reuses the cached llh; three MH blocks each recompute it).

    python tools/bench_gmm.py [--n-log2 20] [--T 100] [--cpu-n 2048]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1306_5583_b200 as P  # noqa: E402
from paper_1306_5583_b200 import gmm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-log2", type=int, default=20)
    ap.add_argument("--T", type=int, default=100)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--cpu-n", type=int, default=0)
    args = ap.parse_args()
    n, T = 1 << args.n_log2, args.T
    y = gmm.generate_data(1000, 1306)
    out = {"config": "gmm", "N": n, "T": T, "n_data": len(y)}
    runs = []
    for seed in range(args.seeds + 1):  # seed 0 = warm-up
        s = gmm.make_sampler(n, data=y, T=T, seed=1306 + seed)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.initialize()
        s.iterate(T)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ds, ps = s.log_zconst, s.path_log_zconst()
        h = s.history()
        if seed:
            runs.append({"seed": 1306 + seed, "ms": ms, "log_z_ds": ds, "log_z_ps": ps,
                         "resamples": int(sum(h["resampled"])),
                         "acc_rate_mu": float(sum(h["accept.1"]) / (n * T))})
    ms = min(r["ms"] for r in runs) if runs else float("nan")
    out["runs"] = runs
    out["ms_per_run"] = ms
    out["particle_iterations_per_s"] = n * T / (ms * 1e-3)
    llh_evals = n * (1 + 3 * T) * len(y) * gmm.R
    out["component_evals_per_s"] = llh_evals / (ms * 1e-3)
    if args.cpu_n:
        from oracle import oracle as O
        h5 = gmm.default_hyper(y)
        th = os.cpu_count() or 1
        t0 = time.perf_counter()
        ref = O.gmm_run(args.cpu_n, 1307, "stratified", 0.5, y, h5, T, 2.0, r=gmm.R, nthreads=th)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": args.cpu_n * T / dt, "unit": "particle-iterations/s", "cores": th,
                               "kind": "port", "sample": f"oracle orc_gmm_run N={args.cpu_n} T={T}",
                               "log_z_ds": float(ref[-1, 7])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
