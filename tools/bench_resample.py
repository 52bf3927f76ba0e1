"""Config 5: resample + copy microbenchmark, N = 2^10 .. 2^30, all six schemes,
uniform / skewed / degenerate weights (BASELINE.json configs[4]).

One call = smc_resample on normalized W (HBM) with uniforms drawn on the device
from the resampling stream, counts + parent map, and the in-place copy of every
zero-count 32-byte state row.  Algorithmic bytes:
    N * (8 W + 4 counts + 4 parents) + 64 * (#rows with parents[j] != j).
Timed with CUDA events over `reps` calls after warm-up; inputs > L2 from 2^24 up.

    python tools/bench_resample.py [--max-log2 30] [--out profiles/r1_resample_microbench.jsonl]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1306_5583_b200 as P  # noqa: E402
from paper_1306_5583_b200 import _abi  # noqa: E402

SCHEMES = ["systematic", "stratified", "multinomial", "residual", "residual_stratified", "residual_systematic"]


def weights(n, kind, g):
    if kind == "uniform":
        lw = (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5) * 2e-3
    elif kind == "skewed1":
        lw = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    elif kind == "skewed3":
        lw = 3 * torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    else:  # degenerate
        lw = torch.full((n,), -50.0, dtype=torch.float64, device="cuda")
        lw[0] = 0.0
    w = torch.exp(lw - lw.max())
    return (w / w.sum()).contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--step", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--schemes", default=",".join(SCHEMES))
    ap.add_argument("--kinds", default="uniform,skewed1,skewed3,degenerate")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6543.4
    g = torch.Generator(device="cuda")
    g.manual_seed(1306)
    lines = []
    for lg in range(args.min_log2, args.max_log2 + 1, args.step):
        n = 1 << lg
        x = torch.randn((n, 4), dtype=torch.float64, device="cuda", generator=g)
        counts = torch.empty(n, dtype=torch.int32, device="cuda")
        parents = torch.empty(n, dtype=torch.int32, device="cuda")
        ws = torch.empty(_abi.lib().smc_resample_workspace_bytes(n), dtype=torch.uint8, device="cuda")
        status = torch.zeros(3, dtype=torch.int32, device="cuda")  # smc_status
        rng = P.RngStreamSet(n + 1, 1306)
        kinds = args.kinds.split(",")
        for kind in kinds:
            w = weights(n, kind, g)
            for scheme in args.schemes.split(","):
                sid = int(P.ResampleScheme[scheme.title().replace("_", "")])

                def call():
                    _abi.call("smc_resample", sid, ctypes.c_void_p(w.data_ptr()), None, None, n, n, rng.seed, n,
                              rng.counter_ptr(n), None, 0, ctypes.c_void_p(counts.data_ptr()),
                              ctypes.c_void_p(parents.data_ptr()), ctypes.c_void_p(x.data_ptr()), 32, None,
                              ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                              _abi.stream())
                reps = 20 if lg <= 24 else 5
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                assert int(status[0].item()) == 0
                ms = e0.elapsed_time(e1) / reps
                moved = int((parents != torch.arange(n, device="cuda", dtype=torch.int32)).sum().item())
                byts = n * 16 + 64 * moved
                d = {"n": n, "log2n": lg, "scheme": scheme, "weights": kind, "ms": ms, "moved_frac": moved / n,
                     "alg_bytes": byts, "GBps": byts / (ms * 1e-3) / 1e9, "frac_of_hbm": byts / (ms * 1e-3) / 1e9 / peak,
                     "Mparticles_per_s": n / (ms * 1e-3) / 1e6}
                lines.append(d)
                print(json.dumps(d), flush=True)
        del x, counts, parents, ws, rng
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for d in lines:
                f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
