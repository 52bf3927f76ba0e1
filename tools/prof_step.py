"""Small driver for ncu: PF at N (default 2^24), init + W+K steps, no timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1306_5583_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
scheme = sys.argv[3] if len(sys.argv) > 3 else "systematic"
obs = np.cumsum(np.random.default_rng(1306).normal(0, 0.15, (100, 2)), 0)
s = P.pf.make_sampler(n, scheme, 0.5, seed=1306)
s.initialize(obs)
s.iterate(steps)
torch.cuda.synchronize()
print("ok", s.history()["ess_over_n"][-1])
