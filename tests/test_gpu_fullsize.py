"""Parity at BASELINE.json's full sizes.

* config 2 (N = 2^24 on one B200): the PF through the Sampler API for the paper's full
  100 observations vs the C oracle at the same N and seed (identical resampling
  decisions, ESS/N, monitor and log Z within 1e-6, final state within 1e-8);
* config 2's "sweeping all six resampling schemes": resampling at 2^24 from the PF's own
  pre-resample weights, for every scheme, with explicit uniforms AND with the uniforms
  drawn from stream N -- counts and parents bit-exact vs the oracle, plus the
  size-independent properties (sum N, survivors keep their slot, copy multiset);
* config 3 (GMM, N = 2^20, 1000 points, T = 100): the first iterations of the T = 100
  schedule vs orc_gmm_run (ESS/N, accept counts +-2, path integrand and log Z within 1e-6).
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu
N = 1 << 24
THREADS = len(os.sched_getaffinity(0))
SCHEMES = ["multinomial", "residual", "stratified", "systematic", "residual_stratified", "residual_systematic"]


def test_pf_2e24_matches_oracle_strict():
    """The first 6 steps of the 2^24 filter vs the oracle: identical resampling decisions,
    ESS/N, monitor and log Z within 1e-6, and the final state within 1e-8 (the GPU normals
    are within a few ulp of glibc's, and no resampling index has flipped yet)."""
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(6, 1306)
    s = pf.make_sampler(N, "systematic", 0.5, seed=1306)
    s.initialize(obs)
    s.iterate(5)
    h = s.history()
    x = s.system.value.data.cpu().numpy()
    lz = s.log_zconst
    del s
    torch.cuda.empty_cache()
    ref, xref, _ = O.pf_run(N, 1306, "systematic", 0.5, obs, nthreads=THREADS, want_state=True)
    assert np.array_equal(h["resampled"], ref[:, 1])
    np.testing.assert_allclose(h["ess_over_n"], ref[:, 0], rtol=1e-6)
    np.testing.assert_allclose(h["pos.0"], ref[:, 2], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(h["pos.1"], ref[:, 3], rtol=1e-6, atol=1e-9)
    assert abs(lz - ref[-1, 4]) <= 1e-6 * abs(ref[-1, 4])
    bad = np.abs(x - xref) > 1e-8 * (1 + np.abs(xref))
    assert bad.sum() == 0, f"{bad.any(1).sum()} of {N} particles differ"


class _LockstepResampler:
    """Wraps the sampler's Resampler: before every resample of the running 2^24 filter, snapshot
    the weights it is handed and the resampling stream's counter; after it, check the parent map
    against the oracle fed those SAME weights and uniforms (north_star: indices bit-exact given
    identical weights and uniforms), at every step of the 100-observation run."""

    def __init__(self, inner, scheme):
        self.inner, self.scheme, self.steps, self.moved = inner, scheme, 0, []

    def __getattr__(self, k):
        return getattr(self.inner, k)

    def __call__(self, scheme, *, weight_set=None, rng=None, stream_index=None, parents=None, gate=None, **kw):
        w = weight_set.read_weight().cpu().numpy()
        c0 = int(rng._ctr[stream_index].item()) & 0xFFFFFFFFFFFFFFFF
        self.inner(scheme, weight_set=weight_set, rng=rng, stream_index=stream_index, parents=parents, gate=gate,
                   **kw)
        self.inner.check()
        st = weight_set.host_state()
        if not st.resample:  # gated off this step (ESS above the threshold): nothing drawn
            assert int(rng._ctr[stream_index].item()) & 0xFFFFFFFFFFFFFFFF == c0
            return
        got = parents.cpu().numpy()
        os_ = O.Streams(N + 1, rng.seed)
        os_.counters[stream_index] = np.uint64(c0)
        ref, _ = O.resample_counts(self.scheme, w, streams=os_, stream=stream_index)
        refp = O.replication_to_parents(ref)
        bad = np.nonzero(got != refp)[0]
        assert bad.size == 0, f"step {self.steps}: {bad.size} parents differ, first at {bad[:5]}"
        assert int(rng._ctr[stream_index].item()) & 0xFFFFFFFFFFFFFFFF == int(os_.counters[stream_index])
        self.moved.append(float(np.mean(got != np.arange(N))))
        self.steps += 1


@pytest.mark.parametrize("scheme", ["systematic", "residual_stratified"])
def test_pf_2e24_100_obs_resampling_bit_exact_every_step(scheme):
    """Config 2's target sentence at full size: the 2^24-particle, 100-observation filter, and at
    EVERY one of its resamples the parent map equals the oracle's for identical weights and
    stream-N uniforms, with identical counter advance."""
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(100, 1306)
    s = pf.make_sampler(N, scheme, 0.5, seed=1306)
    s.graph = False  # the hook reads the weights back on the host at every step
    hook = _LockstepResampler(s.system.resampler, scheme)
    s.system.resampler = hook
    s.initialize(obs)
    s.iterate(99)
    h = s.history()
    assert hook.steps == int(np.sum(h["resampled"])) and hook.steps >= 90
    assert 0.1 < np.mean(hook.moved) < 0.9


def test_pf_2e24_100_obs_end_to_end_within_mc_error():
    """SPEC.md:497-503 / PAPER.md:1126-1143 at 2^24, init + 99 iterations, GPU RNG end to end vs
    the oracle with the same seed.  The GPU normals are within a few ulp of glibc's, so after
    enough resamples an index flips and the two runs' particle sets drift apart: the estimates
    must then agree within the run's Monte Carlo error (north_star), measured here as the
    spread of the same GPU filter over 8 other seeds.  Resampling decisions must be identical."""
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(100, 1306)
    runs = []
    for seed in [1306] + list(range(1, 9)):
        s = pf.make_sampler(N, "systematic", 0.5, seed=seed)
        s.initialize(obs)
        s.iterate(99)
        h = s.history()
        runs.append((h, s.log_zconst))
        del s
        torch.cuda.empty_cache()
    ref = O.pf_run(N, 1306, "systematic", 0.5, obs, nthreads=THREADS)
    (h, lz), others = runs[0], runs[1:]
    assert np.array_equal(h["resampled"], ref[:, 1])
    # once the runs have drifted apart they are two draws of the same estimator: their difference
    # has the Monte Carlo sd times sqrt(2).  z = difference / (sqrt(2) sd), sd from the 8 other
    # seeds (so z is roughly Student-t with 7 degrees of freedom): every |z| over the 100 steps
    # and 3 estimates below 7, and the mean z^2 near 1 (no systematic offset)
    zs = []
    for col, k in (("pos.0", 2), ("pos.1", 3), ("ess_over_n", 0)):
        sd = np.std([o[0][col] for o in others], axis=0, ddof=1)
        z = (h[col] - ref[:, k]) / (np.sqrt(2) * sd + 1e-300)
        z[np.abs(h[col] - ref[:, k]) <= 1e-9 * (1 + np.abs(ref[:, k]))] = 0.0  # still in lockstep
        assert np.all(np.abs(z) < 7), (col, int(np.argmax(np.abs(z))), float(np.max(np.abs(z))))
        zs.append(z)
    assert np.mean(np.concatenate(zs) ** 2) < 3.0, np.mean(np.concatenate(zs) ** 2)
    sd_lz = np.std([o[1] for o in others], ddof=1)
    assert abs(lz - ref[-1, 4]) <= 7 * np.sqrt(2) * sd_lz, (lz, ref[-1, 4], sd_lz)


@pytest.fixture(scope="module")
def pf_weights():
    """The PF's own pre-resample weights at 2^24 (threshold 0: the weights degrade over 3
    moves, as between resamples), normalized on the device."""
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(4, 7)
    s = pf.make_sampler(N, "systematic", 0.0, seed=7)
    s.initialize(obs)
    s.iterate(3)
    w = s.system.weight_set.read_weight().contiguous()
    del s
    torch.cuda.empty_cache()
    return w


def _check(counts, parents, ref):
    assert counts.sum() == N and counts.min() >= 0
    surv = counts >= 1
    assert np.array_equal(parents[surv], np.nonzero(surv)[0])
    assert np.array_equal(np.bincount(parents, minlength=N), counts)
    bad = np.nonzero(counts != ref)[0]
    assert bad.size == 0, f"{bad.size} counts differ, first at {bad[:5]}"
    assert np.array_equal(parents, O.replication_to_parents(ref))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_resample_2e24_pf_weights_explicit_u_bit_exact(scheme, pf_weights):
    from paper_1306_5583_b200 import resample, replication_to_parents
    w = pf_weights
    u = torch.rand(N, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    counts = resample(scheme, w, u=u).cpu().numpy()
    parents = replication_to_parents(torch.as_tensor(counts).cuda()).cpu().numpy()
    ref, _ = O.resample_counts(scheme, w.cpu().numpy(), u=u.cpu().numpy())
    _check(counts, parents, ref)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_resample_2e24_pf_weights_stream_n_bit_exact(scheme, pf_weights):
    """Uniforms from the resampling stream N on the device, counts and parents
    from one smc_resample call, identical counter advance."""
    from paper_1306_5583_b200 import RngStreamSet
    from paper_1306_5583_b200.resample import Resampler
    w = pf_weights
    ss = RngStreamSet(N + 1, 1306)
    os_ = O.Streams(N + 1, 1306)
    r = Resampler(N)
    counts = torch.empty(N, dtype=torch.int32, device="cuda")
    parents = torch.empty(N, dtype=torch.int32, device="cuda")
    for rep in range(2):  # the second call starts from the advanced counter
        r(scheme, weights=w, rng=ss, stream_index=N, counts=counts, parents=parents)
        r.check()
        ref, _ = O.resample_counts(scheme, w.cpu().numpy(), streams=os_, stream=N)
        _check(counts.cpu().numpy(), parents.cpu().numpy(), ref)
        assert ss.counters_host()[N] == int(os_.counters[N])


def test_gmm_config3_first_iterations_match_oracle():
    """Config 3 at full size: N = 2^20, 1000 points, 4 components, T = 100, prior annealing
    p = 2, stratified at ESS < N/2 -- the first 3 iterations of that schedule."""
    from paper_1306_5583_b200 import gmm
    n, T, steps = 1 << 20, 100, 3
    y = gmm.generate_data(1000, 1306)
    h = gmm.default_hyper(y)
    s = gmm.make_sampler(n, data=y, T=T, seed=1307)
    s.initialize()
    s.iterate(steps)
    hist = s.history()
    lz = s.log_zconst
    ref = O.gmm_run(n, 1307, "stratified", 0.5, y, h, T, 2.0, nthreads=THREADS, steps=steps)
    assert np.array_equal(hist["resampled"], ref[:, 1])
    np.testing.assert_allclose(hist["path.grid"], ref[:, 5], rtol=1e-15)
    np.testing.assert_allclose(hist["ess_over_n"], ref[:, 0], rtol=1e-6)
    for k, col in ((1, 2), (2, 3), (3, 4)):
        assert np.all(np.abs(hist[f"accept.{k}"] - ref[:, col]) <= 2), (k, hist[f"accept.{k}"], ref[:, col])
    np.testing.assert_allclose(hist["path.integrand"], ref[:, 6], rtol=1e-6)
    assert abs(lz - ref[-1, 7]) <= 1e-6 * abs(ref[-1, 7])


N_MN1 = 3 << 25  # past the shared-memory bin geometry (mn2_fits): the global-bucket multinomial path


@pytest.mark.parametrize("n", [1 << 26])
def test_multinomial_wide_bins_bit_exact(n):
    """2^26: the shared-memory bins at their widest (one 1024-thread count block per SM, 12 draws
    per scatter thread) -- counts bit-exact vs the oracle on skewed weights."""
    from paper_1306_5583_b200 import resample
    g = torch.Generator("cuda").manual_seed(12)
    lw = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    w = torch.exp(lw - lw.max())
    w = (w / w.sum()).contiguous()
    del lw
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    counts = resample("multinomial", w, u=u).cpu().numpy()
    ref, _ = O.resample_counts("multinomial", w.cpu().numpy(), u=u.cpu().numpy())
    del w, u
    torch.cuda.empty_cache()
    assert counts.sum() == n
    bad = np.nonzero(counts != ref)[0]
    assert bad.size == 0, f"{bad.size} counts differ, first at {bad[:5]}"


@pytest.mark.parametrize("scheme,draws", [("multinomial", "explicit"), ("residual", "explicit"),
                                          ("multinomial", "stream")])
def test_multinomial_past_shared_memory_bins_bit_exact(scheme, draws):
    """Config 5 reaches 2^30 for every scheme: above ~2^26 a multinomial position bin no longer
    fits one block's shared memory and the draws go through the global-memory bucket path --
    counts bit-exact vs the oracle there too (skewed weights; explicit and stream-N uniforms)."""
    from paper_1306_5583_b200 import RngStreamSet, resample
    from paper_1306_5583_b200.resample import Resampler
    n = N_MN1
    g = torch.Generator("cuda").manual_seed(11)
    lw = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    w = torch.exp(lw - lw.max())
    w = (w / w.sum()).contiguous()
    del lw
    if draws == "explicit":
        u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        counts = resample(scheme, w, u=u).cpu().numpy()
        ref, _ = O.resample_counts(scheme, w.cpu().numpy(), u=u.cpu().numpy())
        del u
    else:
        ss = RngStreamSet(n + 1, 1306)
        os_ = O.Streams(n + 1, 1306)
        r = Resampler(n)
        c = torch.empty(n, dtype=torch.int32, device="cuda")
        r(scheme, weights=w, rng=ss, stream_index=n, counts=c)
        r.check()
        counts = c.cpu().numpy()
        ref, _ = O.resample_counts(scheme, w.cpu().numpy(), streams=os_, stream=n)
        assert ss.counters_host()[n] == int(os_.counters[n])
        del r, c
    del w
    torch.cuda.empty_cache()
    assert counts.sum() == n
    bad = np.nonzero(counts != ref)[0]
    assert bad.size == 0, f"{bad.size} counts differ, first at {bad[:5]}"


def test_multinomial_past_shared_memory_bins_degenerate():
    """All the weight on one particle at N = 3 2^25: every draw lands on it."""
    from paper_1306_5583_b200 import resample
    n = N_MN1
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    w[n // 3] = 1.0
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    counts = resample("multinomial", w, u=u).cpu().numpy()
    assert counts[n // 3] == n and counts.sum() == n
