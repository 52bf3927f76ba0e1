import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1306_5583_b200 as P
obs, _ = P.pf.generate_observations(100, 1306)
s = P.pf.make_sampler(10000, "systematic", 0.5, seed=1)
s.graph = False
s.initialize(obs)
s.iterate(10)
torch.cuda.synchronize()
