"""Config 1: the paper's PF at N = 10^4, 100 observations, systematic at ESS < N/2 --
wall time of initialize + 99 iterations through the Sampler API (launch-bound size)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_5583_b200 as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    obs, _ = P.pf.generate_observations(100, 1306)
    out = {"config": "PF config 1", "N": n, "steps": 100}
    for mode in (False, "auto"):
        s = P.pf.make_sampler(n, "systematic", 0.5, seed=1306)
        s.graph = mode
        best, first = None, None
        for rep in range(4):  # rep 0 includes the one-time capture (graph mode)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.initialize(obs)
            s.iterate(99)
            s.flush()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if rep == 0:
                first = dt
            else:
                best = dt if best is None else min(best, dt)
        tag = "graph" if mode else "eager"
        out[tag] = {"seconds": best, "us_per_step": best / 100 * 1e6, "first_run_seconds": first,
                    "particle_steps_per_s": n * 100 / best}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
