"""PF at N = 2^24: ms per step of iterate(K) replayed as a CUDA graph vs launched eagerly
(same kernels, PDL either way); CUDA events around the K steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_5583_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
K = int(sys.argv[2]) if len(sys.argv) > 2 else 600
obs = np.cumsum(np.random.default_rng(1306).normal(0, 0.15, (K * 3 + 20, 2)), 0)
for mode in ("eager", "graph", "eager", "graph"):
    s = P.pf.make_sampler(n, "systematic", 0.5, seed=1306)
    s.graph = "auto" if mode == "graph" else False
    s.initialize(obs)
    s.iterate(K, check=False)  # warm-up (and the one-time capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.iterate(K, check=False)
    e1.record()
    torch.cuda.synchronize()
    s.check()
    print(mode, round(e0.elapsed_time(e1) / K, 4), "ms/step", flush=True)
    del s
    torch.cuda.empty_cache()
