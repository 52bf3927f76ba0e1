"""Same-process A/B of the PF move kernels at N = 2^24 (SMC_DEBUG_MOVE_WS 0 / 1): ms per PF step and
per move (median of per-step CUDA events), alternating the two settings over several rounds."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1306_5583_b200 as P  # noqa: E402
from paper_1306_5583_b200 import _abi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
obs = np.cumsum(np.random.default_rng(1306).normal(0, 0.15, (400, 2)), 0)
res = {0: [], 1: []}
for rnd in range(3):
    for ws in (0, 1):
        _abi.call("smc_debug_set", 2, ws)
        s = P.pf.make_sampler(n, "systematic", 0.5, seed=1306)
        s.graph = False
        s.initialize(obs)
        s.iterate(5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.iterate(100, check=False)
        e1.record()
        torch.cuda.synchronize()
        step = e0.elapsed_time(e1) / 100
        s.timing = {}
        s.iterate(30, check=False)
        torch.cuda.synchronize()
        mv = sorted(a.elapsed_time(b) for a, b in s.timing["move"])
        res[ws].append((round(step, 4), round(mv[len(mv) // 2], 4)))
        del s
        torch.cuda.empty_cache()
print(json.dumps({"single_role": res[0], "warp_specialized": res[1]}))
