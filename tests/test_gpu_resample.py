"""Resampling parity: device counts / parent maps / copies are BIT-EXACT with the oracle
for identical normalized weights and uniforms (north_star), all six schemes."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SCHEMES = ["multinomial", "residual", "stratified", "systematic", "residual_stratified", "residual_systematic"]
SIZES = [1, 2, 3, 7, 100, 2047, 2048, 2049, 4097, 10000, 3 * 2048 + 5, (1 << 17) + 3]


def weights(n, kind, seed=1306):
    rng = np.random.default_rng(seed + n)
    if kind == "uniform":
        lw = rng.uniform(-1e-3, 1e-3, n)
    elif kind == "equal":
        lw = np.zeros(n)
    elif kind == "skewed":
        lw = rng.normal(0, 3, n)
    elif kind == "degenerate":
        lw = np.full(n, -50.0)
        lw[n // 3] = 0.0
    elif kind == "sparse":
        lw = np.where(rng.random(n) < 0.05, rng.normal(0, 1, n), -np.inf)
        lw[0] = 0.0
    elif kind == "one_heavy":
        lw = np.full(n, -np.inf)
        lw[n - 1] = 0.0
    return O.normalize_log(lw)[1]


def gpu_resample(scheme, w, u=None, rng=None, m_out=None, rows=None):
    from paper_1306_5583_b200 import _abi
    from paper_1306_5583_b200.resample import Resampler
    n = len(w)
    r = Resampler(n)
    counts = torch.empty(n, dtype=torch.int32, device="cuda")
    parents = torch.empty(n, dtype=torch.int32, device="cuda") if (m_out is None or m_out == n) else None
    rp = None if rows is None else __import__("ctypes").c_void_p(rows.data_ptr())
    r(scheme, weights=torch.as_tensor(w).cuda(), u=None if u is None else torch.as_tensor(u).cuda(), rng=rng,
      stream_index=None if rng is None else rng.size - 1, m_out=m_out, counts=counts, parents=parents, rows=rp,
      row_bytes=0 if rows is None else rows.shape[1] * 8)
    r.check()
    return counts.cpu().numpy(), (None if parents is None else parents.cpu().numpy())


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("kind", ["uniform", "skewed", "degenerate", "sparse", "equal", "one_heavy"])
def test_counts_parents_bit_exact_explicit_u(scheme, kind):
    for n in SIZES:
        w = weights(n, kind)
        u = np.random.default_rng(n).random(n + 1)
        ref, _ = O.resample_counts(scheme, w, u=u)
        got, par = gpu_resample(scheme, w, u=u)
        assert np.array_equal(got, ref), (scheme, kind, n, np.nonzero(got != ref)[0][:5])
        assert np.array_equal(par, O.replication_to_parents(ref)), (scheme, kind, n)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_stream_uniforms_bit_exact(scheme):
    """Uniforms drawn on the device from stream N == the oracle's draws from rng.py's stream N."""
    from paper_1306_5583_b200 import RngStreamSet
    for n in (5, 4099, 70001):
        w = weights(n, "skewed")
        ss = RngStreamSet(n + 1, 1306 + n)
        os_ = O.Streams(n + 1, 1306 + n)
        for rep in range(3):
            ref, draws = O.resample_counts(scheme, w, streams=os_, stream=n)
            got, par = gpu_resample(scheme, w, rng=ss)
            assert np.array_equal(got, ref), (scheme, n, rep)
            assert ss.counters_host()[n] == int(os_.counters[n])  # same draw count


@pytest.mark.parametrize("scheme", SCHEMES)
def test_large_n_properties(scheme):
    n = 1 << 22
    w = weights(n, "skewed")
    u = np.random.default_rng(5).random(n)
    got, par = gpu_resample(scheme, w, u=u)
    assert got.sum() == n and got.min() >= 0
    surv = got >= 1
    assert np.array_equal(par[surv], np.nonzero(surv)[0])
    assert np.array_equal(np.bincount(par, minlength=n), got)  # multiset implied by counts
    ref, _ = O.resample_counts(scheme, w, u=u)
    assert np.array_equal(got, ref)
    assert np.array_equal(par, O.replication_to_parents(ref))


def test_fused_copy_matches_oracle():
    for n in (3, 2049, 100003):
        for d in (4, 1, 6):
            w = weights(n, "skewed")
            u = np.random.default_rng(1).random(n)
            x = np.random.default_rng(2).normal(size=(n, d))
            xg = torch.as_tensor(x).cuda().contiguous()
            counts, par = gpu_resample("systematic", w, u=u, rows=xg)
            ref = O.copy_rows(x.copy(), O.replication_to_parents(counts))
            assert np.array_equal(xg.cpu().numpy(), ref), (n, d)


def test_spec_examples_on_device():
    for s in SCHEMES:
        c, p = gpu_resample(s, [1.0, 0.0, 0.0], u=[0.5, 0.5, 0.5])
        assert list(c) == [3, 0, 0] and list(p) == [0, 0, 0]
    c, p = gpu_resample("systematic", [0.5, 0.5], u=[0.3])
    assert list(c) == [1, 1]
    for s in ("residual", "residual_stratified", "residual_systematic"):  # floors only (no leftovers)
        c, p = gpu_resample(s, [0.5, 0.3, 0.2], u=[0.0], m_out=10)
        assert list(c) == [5, 3, 2], s
    for s in ("residual", "residual_stratified", "residual_systematic"):  # floors + leftovers, M != N
        w = [0.55, 0.25, 0.2]
        c, _ = gpu_resample(s, w, u=[0.3, 0.7, 0.9], m_out=7)
        ref, _ = O.resample_counts(s, np.array(w), u=np.array([0.3, 0.7, 0.9]), m_out=7)
        assert list(c) == list(ref) and sum(c) == 7, (s, list(c), list(ref))
    from paper_1306_5583_b200 import replication_to_parents
    assert replication_to_parents([2, 0, 1]).tolist() == [0, 0, 2]
    assert replication_to_parents([0, 3, 0]).tolist() == [1, 1, 1]
    assert replication_to_parents([1] * 5).tolist() == list(range(5))


def test_replication_to_parents_large():
    from paper_1306_5583_b200 import replication_to_parents
    rng = np.random.default_rng(9)
    for n in (1, 2048, 2049, 300001):
        counts = rng.multinomial(n, np.full(n, 1.0 / n)).astype(np.int32)
        assert np.array_equal(replication_to_parents(counts).cpu().numpy(), O.replication_to_parents(counts))
    counts = np.zeros(50000, np.int32)
    counts[777] = 50000  # one parent with N children: load-balanced
    assert np.all(replication_to_parents(counts).cpu().numpy() == 777)


def test_errors_surface():
    from paper_1306_5583_b200 import _abi, replication_to_parents
    with pytest.raises(_abi.SmcError):
        gpu_resample("stratified", [0.5, 0.6], u=[0.1, 0.2])
    with pytest.raises(_abi.SmcError):
        gpu_resample("stratified", [0.5, float("nan")], u=[0.1, 0.2])
    with pytest.raises(_abi.SmcError):
        replication_to_parents([2, 2, 0])
    with pytest.raises(_abi.SmcError):
        gpu_resample("stratified", [0.5, 0.5], u=[0.1])  # needs 2 uniforms


@pytest.mark.parametrize("scheme", ["stratified", "systematic", "residual_stratified", "residual_systematic"])
def test_fast_F_path_equals_exact_path(scheme):
    """The fp64 guard-band path of F(X) and the exact 128-bit path give identical counts."""
    from paper_1306_5583_b200 import _abi
    for n in (3, 1000, 65537, 1 << 20):
        for kind in ("skewed", "uniform", "equal"):
            w = weights(n, kind)
            u = np.random.default_rng(n + 1).random(n)
            if kind == "equal":
                u[:] = 1 - 2.0 ** -53  # stresses ties at stratum boundaries
            fast, _ = gpu_resample(scheme, w, u=u)
            _abi.call("smc_debug_set", 1, 1)
            try:
                exact, _ = gpu_resample(scheme, w, u=u)
            finally:
                _abi.call("smc_debug_set", 1, 0)
            assert np.array_equal(fast, exact), (scheme, n, kind)


def test_launch_configuration_invariance_sharded_tiles():
    """Counts for a prefix of tiles don't depend on the tail: integer CDF is associative."""
    n = 5 * 2048
    w = weights(n, "skewed")
    u = np.random.default_rng(3).random(n)
    a, _ = gpu_resample("stratified", w, u=u)
    b, _ = gpu_resample("stratified", w, u=u)
    assert np.array_equal(a, b)  # run-to-run determinism


@pytest.mark.parametrize("scheme", SCHEMES)
def test_unbiasedness_acceptance_1_on_device(scheme):
    """SPEC.md:671 on the device: W = (.05, .15, .3, .5), N = 4, draws from the sampler's
    resampling stream (stream N of RngStreamSet(N + 1)), |mean R_i - N W_i| <= 4 SE.
    20000 replicates (each one smc_resample call; the criterion holds at any count)."""
    from paper_1306_5583_b200 import RngStreamSet
    from paper_1306_5583_b200.resample import Resampler
    W = torch.tensor([0.05, 0.15, 0.3, 0.5], dtype=torch.float64, device="cuda")
    reps = 20000
    rng = RngStreamSet(5, 2024)
    r = Resampler(4)
    out = torch.empty((reps, 4), dtype=torch.int32, device="cuda")
    for k in range(reps):
        r(scheme, weights=W, rng=rng, stream_index=4, counts=out[k])
    r.check()
    acc = out.double().cpu().numpy()
    assert np.all(acc.sum(1) == 4)
    mean, sd = acc.mean(0), acc.std(0) + 1e-12
    assert np.all(np.abs(mean - 4 * W.cpu().numpy()) <= 4 * sd / np.sqrt(reps) + 1e-12), mean
    # and the same stream through the oracle gives the same replicates, bit for bit
    st = O.Streams(5, 2024)
    ref = np.array([O.resample_counts(scheme, W.cpu().numpy(), streams=st, stream=4)[0] for _ in range(200)])
    assert np.array_equal(acc[:200].astype(np.int64), ref)


@pytest.mark.parametrize("scheme", ["systematic", "residual_stratified"])
def test_multichunk_tile_scans_bit_exact(scheme):
    """N > 2^24: more tiles (16391) than one chunk of the single-block scans (passes S and S2
    walk 1024 threads x 8 tiles per chunk), counts / parents / the fused 32-byte row copy
    bit-exact with the oracle."""
    n = (1 << 25) + 12345
    w = weights(n, "skewed")
    u = np.random.default_rng(9).random(n)
    x = None
    if scheme == "systematic":
        x = np.random.default_rng(3).normal(size=(n, 4))
        xg = torch.as_tensor(x).cuda().contiguous()
        got, par = gpu_resample(scheme, w, u=u, rows=xg)
    else:
        got, par = gpu_resample(scheme, w, u=u)
    ref, _ = O.resample_counts(scheme, w, u=u)
    assert np.array_equal(got, ref)
    pref = O.replication_to_parents(ref)
    assert np.array_equal(par, pref)
    if x is not None:
        assert np.array_equal(xg.cpu().numpy(), x[pref])


def test_config4_size_2e28_systematic_bit_exact():
    """BASELINE config 4's whole filter size on one GPU, N = 2^28: systematic counts and the
    parent map bit-exact with the oracle (the largest size the int32 parent vector is used at
    in the benchmarks), plus the size-independent invariants."""
    from paper_1306_5583_b200 import replication_to_parents, resample
    n = 1 << 28
    lw = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(28)) * 2.0
    w = torch.exp(lw - torch.logsumexp(lw, 0))
    w = w / w.sum()
    u = torch.tensor([0.3141592653589793], dtype=torch.float64, device="cuda")
    counts = resample("systematic", w, u=u)
    parents = replication_to_parents(counts)
    c = counts.cpu().numpy()
    p = parents.cpu().numpy()
    assert c.sum() == n and c.min() >= 0
    surv = c >= 1
    assert np.array_equal(p[surv], np.nonzero(surv)[0])
    ref, _ = O.resample_counts("systematic", w.cpu().numpy(), u=u.cpu().numpy())
    assert np.array_equal(c, ref)
    assert np.array_equal(p, O.replication_to_parents(ref))
