"""Parity at BASELINE.json's full size (config 2: N = 2^24 on one B200).

* the PF through the Sampler API for 6 steps vs the C oracle at the same N and seed
  (identical resampling decisions, ESS/N, monitor and log Z within 1e-6, final state 1e-8);
* resampling at 2^24 from the PF's own pre-resample weights: counts and parents bit-exact,
  plus the size-independent properties (sum N, survivors keep their slot, copy multiset).
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu
N = 1 << 24
THREADS = len(os.sched_getaffinity(0))


def test_pf_2e24_matches_oracle():
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(6, 1306)
    s = pf.make_sampler(N, "systematic", 0.5, seed=1306)
    s.initialize(obs)
    s.iterate(5)
    h = s.history()
    ref, xref, lwref = O.pf_run(N, 1306, "systematic", 0.5, obs, nthreads=THREADS, want_state=True)
    assert np.array_equal(h["resampled"], ref[:, 1])
    np.testing.assert_allclose(h["ess_over_n"], ref[:, 0], rtol=1e-6)
    np.testing.assert_allclose(h["pos.0"], ref[:, 2], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(h["pos.1"], ref[:, 3], rtol=1e-6, atol=1e-9)
    assert abs(s.log_zconst - ref[-1, 4]) <= 1e-6 * abs(ref[-1, 4])
    x = s.system.value.data.cpu().numpy()
    bad = np.abs(x - xref) > 1e-8 * (1 + np.abs(xref))
    assert bad.sum() == 0, f"{bad.any(1).sum()} of {N} particles differ"


@pytest.mark.parametrize("scheme", ["systematic", "stratified", "residual_systematic"])
def test_resample_2e24_pf_weights_bit_exact(scheme):
    from paper_1306_5583_b200 import pf, resample, replication_to_parents
    obs, _ = pf.generate_observations(3, 7)
    s = pf.make_sampler(N, "systematic", 0.0, seed=7)  # threshold 0: no resampling, weights degrade
    s.initialize(obs)
    s.iterate(2)
    w = s.system.weight_set.read_weight()
    u = torch.rand(N, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    counts = resample(scheme, w, u=u).cpu().numpy()
    parents = replication_to_parents(torch.as_tensor(counts).cuda()).cpu().numpy()
    assert counts.sum() == N and counts.min() >= 0
    surv = counts >= 1
    assert np.array_equal(parents[surv], np.nonzero(surv)[0])
    assert np.array_equal(np.bincount(parents, minlength=N), counts)
    ref, _ = O.resample_counts(scheme, w.cpu().numpy(), u=u.cpu().numpy())
    assert np.array_equal(counts, ref)
    assert np.array_equal(parents, O.replication_to_parents(ref))
