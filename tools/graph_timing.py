import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_1306_5583_b200 as P
from paper_1306_5583_b200 import core
obs, _ = P.pf.generate_observations(100, 1306)
s = P.pf.make_sampler(10000, "systematic", 0.5, seed=1)
s.initialize(obs)
s.iterate(3, check=False); torch.cuda.synchronize()
orig = torch.cuda.CUDAGraph.capture_end
def timed_end(self):
    t0 = time.perf_counter(); orig(self); torch.cuda.synchronize(); print("capture_end (instantiate)", time.perf_counter() - t0)
torch.cuda.CUDAGraph.capture_end = timed_end
ob = torch.cuda.CUDAGraph.capture_begin
def timed_begin(self, *a, **k):
    global tb; tb = time.perf_counter(); ob(self, *a, **k)
torch.cuda.CUDAGraph.capture_begin = timed_begin
t0 = time.perf_counter(); s.iterate(10, check=False); torch.cuda.synchronize(); print("iterate(10) incl capture", time.perf_counter() - t0)
t0 = time.perf_counter(); s.iterate(10, check=False); torch.cuda.synchronize(); print("iterate(10) replay", time.perf_counter() - t0)
