"""Drive every kernel of libsmcb200.so at small N, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_run.py

Covers: RNG fills / per-stream draws, every WeightSet mode, all six resampling
schemes (counts, parent map, fused 32-byte row copy, the separate copy for other
row sizes), replication_to_parents, gather / in-place copies, the PF sampler
(counter-array and uniform-count moves, the fused monitor, a CUDA-graph replay),
the GMM sampler (init, reweight, the three MH blocks, path), a run-time compiled
user kernel, and the sharded resample (2 ranks emulated by threads on one GPU).
Exit code 0 when every check passes; the sanitizer reports its own errors.
"""

import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1306_5583_b200 as P  # noqa: E402
from paper_1306_5583_b200 import gmm, pf  # noqa: E402
from paper_1306_5583_b200.resample import Resampler  # noqa: E402

SCHEMES = ["multinomial", "residual", "stratified", "systematic", "residual_stratified", "residual_systematic"]


def rng_and_weights(n):
    rs = P.RngStreamSet(n + 1, 1306)
    st = rs.stream(n)
    st.uniform01(1000)
    st.normal(0.0, 1.0, 1000)
    st.gamma(2.0, 1.0, 50)
    w = P.WeightSet(n)
    v = torch.randn(n, dtype=torch.float64, device="cuda")
    w.set_log_weight(v)
    w.add_log_weight(v * 0.5, accumulate_nc=True)
    w.set_weight(torch.rand(n, dtype=torch.float64, device="cuda") + 0.1)
    w.mul_weight(torch.rand(n, dtype=torch.float64, device="cuda") + 0.1)
    w.set_equal_weight()
    w.read_weight()
    w.read_log_weight()
    return rs


def resampling(n):
    rs = P.RngStreamSet(n + 1, 7)
    lw = torch.randn(n, dtype=torch.float64, device="cuda") * 2
    w = torch.softmax(lw, 0).contiguous()
    for name in SCHEMES:
        r = Resampler(n)
        counts = torch.empty(n, dtype=torch.int32, device="cuda")
        parents = torch.empty(n, dtype=torch.int32, device="cuda")
        x4 = torch.randn(n, 4, dtype=torch.float64, device="cuda")
        import ctypes
        r(name, weights=w, rng=rs, counts=counts, parents=parents, rows=ctypes.c_void_p(x4.data_ptr()), row_bytes=32)
        x3 = torch.randn(n, 3, dtype=torch.float64, device="cuda")
        r(name, weights=w, rng=rs, counts=counts, parents=parents, rows=ctypes.c_void_p(x3.data_ptr()), row_bytes=24)
        r(name, weights=w, u=torch.rand(n, dtype=torch.float64, device="cuda"), counts=counts)
        r.check()
        par = P.replication_to_parents(counts)
        assert int(counts.sum()) == n and par.shape[0] == n
    sm = P.StateMatrix(n, 3)
    sm.data.copy_(torch.randn(n, 3, dtype=torch.float64, device="cuda"))
    sm.copy_particles(torch.randint(0, n, (n,), device="cuda"))


def pf_runs(n):
    obs, _ = pf.generate_observations(80, 1306)
    for scheme in ("systematic", "multinomial", "residual"):
        s = pf.make_sampler(n, scheme, 0.5, seed=3)
        s.graph_min_steps = 4
        s.initialize(obs)
        s.iterate(3)
        _ = s.system.rng_set.counters  # the counter-array move from here on
        s.graph = False
        s.iterate(2)
        s.graph = "auto"
        s.iterate(10)  # CUDA-graph replay
        s.history()


def gmm_runs(n):
    y = gmm.generate_data(100, 1306)
    s = gmm.make_sampler(n, data=y, T=4, seed=1)
    s.initialize()
    s.iterate(4)
    s.path_log_zconst()
    s2 = gmm.make_sampler(n, data=y, T=3, seed=2, components=2)
    s2.initialize()
    s2.iterate(3)


def user_kernel(n):
    from test_gpu_user import _user_pf
    obs, _ = pf.generate_observations(6, 7)
    s = _user_pf(n, "systematic", 1306, obs)
    s.initialize()
    s.iterate(4)
    s.history()


def sharded(n, G=2):
    from test_gpu_dist_sampler import ThreadComm, _run_rank
    obs, _ = pf.generate_observations(8, 1306)
    shared = ThreadComm(G)
    out, errs = [None] * G, []
    th = [threading.Thread(target=_run_rank, args=(shared, r, n, obs, 6, "systematic", out, errs)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def main():
    torch.cuda.set_device(0)
    n = int(os.environ.get("SAN_N", "4099"))
    for name, fn in (("rng+weights", rng_and_weights), ("resampling", resampling), ("pf", pf_runs),
                     ("gmm", gmm_runs), ("user", user_kernel), ("sharded", sharded)):
        fn(n)
        torch.cuda.synchronize()
        print(f"sanitize_run: {name} ok (N={n})", flush=True)


if __name__ == "__main__":
    main()
