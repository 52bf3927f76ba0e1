"""Same-box A/B of the PF move: smc_pf_move_uniform (streams at one count) vs smc_pf_move
(counter array), N = 2^24, median of per-launch CUDA-event times over 200 moves each."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1306_5583_b200 import pf

n = 1 << 24
rs = np.random.default_rng(1306)
obs = np.cumsum(rs.normal(0, 0.15, (1000, 2)), 0)
s = pf.make_sampler(n, "systematic", -1.0, seed=1306)  # no resampling: plain moves
s.initialize(obs)
res = {"uniform": [], "array": []}
for rep in range(400):
    mode = "uniform" if rep % 2 == 0 else "array"
    if mode == "array":
        s.system.rng_set.counters  # drop the uniform-count knowledge for this move
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.move_queue[0](s.iteration + 1, s.system)
    e1.record()
    torch.cuda.synchronize()
    s.iteration += 1
    if mode == "array":  # the array is now current: every stream at the same count again
        v = int(s.system.rng_set._ctr[0].item()) % (1 << 64)
        s.system.rng_set.advance_uniform(n, v, True)
    if rep >= 20:
        res[mode].append(e0.elapsed_time(e1))
print("  ".join(f"{k} median {np.median(v):.4f} ms min {np.min(v):.4f} ms (n={len(v)})" for k, v in res.items()))
