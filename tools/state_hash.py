"""Hash of a short PF run's particle state and log-weights (A/B of library variants that must be
bit-identical): python tools/state_hash.py [N] [steps].  Uses whatever SMC_LIB_PATH selects."""
import hashlib
import sys

import paper_1306_5583_b200 as smc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
obs, _ = smc.pf.generate_observations(100, seed=1306)
s = smc.pf.make_sampler(n, "systematic", 0.5, seed=1306)
s.initialize(obs)
s.iterate(steps)
h = hashlib.sha256()
h.update(s.system.value.data.cpu().numpy().tobytes())
h.update(s.system.weight_set.read_log_weight().cpu().numpy().tobytes())
h.update(repr(s.log_zconst).encode())
print(h.hexdigest()[:16])
