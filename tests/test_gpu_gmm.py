"""GMM SMC sampler (config 3): device kernels vs the oracle,
SPEC.md's examples and invariants, and acceptance criteria 4 and 5."""

import ctypes
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _eval(rows, y, h, r=4):
    from paper_1306_5583_b200 import _abi
    h = list(h) + [0.0] * (6 - len(h))
    x = torch.as_tensor(np.asarray(rows, np.float64).reshape(-1, 16)).cuda().contiguous()
    yy = torch.as_tensor(np.asarray(y, np.float64)).cuda()
    _abi.call("smc_gmm_eval", _abi.ptr(x), x.shape[0], r, _abi.ptr(yy), yy.numel(), (ctypes.c_double * 6)(*h),
              _abi.stream())
    return x.cpu().numpy()


def _row(mu, lam, om):
    r = np.zeros(16)
    r[0:len(mu)], r[4:4 + len(lam)], r[8:8 + len(om)] = mu, lam, om
    return r


def test_llh_spec_examples():
    h = [0.0, 1.0, 2.0, 1.0, 1.0]
    out = _eval([_row([0], [1], [1])], [0.0], h, r=1)
    assert abs(out[0, 13] - (-0.5 * math.log(2 * math.pi))) < 2e-16  # SPEC.md:538 (-0.918939)
    y = np.linspace(-2, 2, 17)
    one = _eval([_row([0.7], [2], [1])], y, h, r=1)[0, 13]
    two = _eval([_row([0.7, 0.7], [2, 2], [0.5, 0.5])], y, h, r=2)[0, 13]
    assert abs(one - two) < 1e-12  # identical components collapse
    # brute-force density sum without the log-lambda cache
    rw = _row([-1, 0.5, 2, 4], [0.5, 2, 1, 3], [0.1, 0.2, 0.3, 0.4])
    dens = sum(math.log(sum(w * math.sqrt(l / (2 * math.pi)) * math.exp(-0.5 * l * (yk - m) ** 2)
                            for m, l, w in zip(rw[0:4], rw[4:8], rw[8:12]))) for yk in y)
    assert abs(_eval([rw], y, h)[0, 13] - dens) < 1e-11
    assert abs(_eval([rw], y, h)[0, 13] - O.gmm_llh(rw, y)) < 1e-11


@pytest.mark.parametrize("r", [1, 2, 3, 4])
def test_prior_spec_examples(r):
    h = [1.5, 0.25, 2.0, 3.0, 1.0]
    row = _row([1.5] * r, [1.0] * r, [1.0 / r] * r)
    out = _eval([row], [0.0], h, r=r)
    gam = r * ((2 - 1) * math.log(1.0) - 1.0 / 3.0 - math.lgamma(2.0) - 2 * math.log(3.0))
    expect = r * 0.5 * math.log(0.25 / (2 * math.pi)) + gam + math.log(math.factorial(r - 1))
    assert abs(out[0, 12] - expect) < 1e-12
    assert abs(out[0, 12] - O.gmm_lprior(row, h, r)) < 1e-12
    h2 = [0.3, 0.5, 3.0, 0.7, 2.5]
    row2 = _row([0.1, -2, 5, 1][:r], [0.5, 2, 1, 3][:r], ([0.1, 0.2, 0.3, 0.4][:r] if r > 1 else [1.0]))
    assert abs(_eval([row2], [0.0], h2, r=r)[0, 12] - O.gmm_lprior(row2, h2, r)) < 1e-12
    hk = h2 + [4.0]  # lambda known: no Gamma term
    assert abs(_eval([row2], [0.0], hk, r=r)[0, 12] - O.gmm_lprior(row2, hk, r)) < 1e-12


def test_scales_and_schedules():
    from paper_1306_5583_b200 import gmm
    a = 0.5
    assert abs((1 + math.sqrt(1 / a)) * 0.15 - 0.362132) < 1e-6 and abs(0.15 / a - 0.3) < 1e-15
    assert abs((1 + math.sqrt(1 / a)) * 0.2 - 0.482843) < 1e-6
    lin, pri = gmm.alpha_linear(10), gmm.alpha_prior(10, 2.0)
    assert lin(0) == 0 and lin(10) == 1 and pri(5) == 0.25
    v = gmm.GmmState(4)
    v.set_alpha(0.01)
    v.set_alpha(1.5)
    assert v.alpha == 1.0 and abs(v.alpha_inc - 0.99) < 1e-15  # clamp


@pytest.mark.parametrize("r,lam_known", [(4, 0.0), (2, 0.0), (1, 0.0), (1, 2.0), (3, 1.5)])
def test_init_and_mh_match_oracle(r, lam_known):
    from paper_1306_5583_b200 import gmm
    n = 2000
    y = gmm.generate_data(200, 7)
    h = gmm.default_hyper(y, lam_known)
    s = gmm.make_sampler(n, data=y, T=10, seed=99, hyper=h, components=r)
    s.initialize()
    v = s.system.value
    x = v.data.cpu().numpy()
    st = O.Streams(n + 1, 99)
    xo = O.gmm_init(n, st, y, h, r)
    np.testing.assert_allclose(x, xo, rtol=1e-12, atol=1e-12)
    assert s.system.rng_set.counters_host()[:n] == [int(c) for c in st.counters[:n]]
    assert np.all(np.abs(x[:, 8:8 + r].sum(1) - 1) < 1e-14)
    v.alpha = 0.3
    v.sds = (0.5, 0.4, 0.6)
    for block, op in ((0, gmm.gmm_move_mu()), (1, gmm.gmm_move_lambda()), (2, gmm.gmm_move_weight())):
        before = v.data.clone()
        acc = int(op.kernel(1, s.system).item())
        acc_o = O.gmm_mh(block, xo, st, y, h, 0.3, v.sds[block], r)
        assert acc == acc_o
        after = v.data
        np.testing.assert_allclose(after.cpu().numpy(), xo, rtol=1e-11, atol=1e-11)
        # MH rollback: rejected rows are bit-identical to their pre-proposal snapshot
        changed = (after != before).any(dim=1)
        assert int(changed.sum()) <= acc
    # cache coherence: recomputing from scratch matches the caches to 1e-10
    cur = v.data.cpu().numpy()
    fresh = _eval(cur, y, h, r)
    np.testing.assert_allclose(fresh[:, 12:14], cur[:, 12:14], rtol=1e-10, atol=1e-10)


def test_zero_scale_always_accepts():
    from paper_1306_5583_b200 import gmm
    n = 1024
    s = gmm.make_sampler(n, data=gmm.generate_data(50, 3), T=10, seed=4)
    s.initialize()
    v = s.system.value
    v.alpha, v.sds = 0.7, (0.0, 0.0, 0.0)
    before = v.data.clone()
    for op in (gmm.gmm_move_mu(), gmm.gmm_move_lambda()):
        assert int(op.kernel(1, s.system).item()) == n
    assert torch.equal(v.data, before)


def test_full_run_matches_oracle():
    from paper_1306_5583_b200 import gmm
    n, T = 4096, 30
    y = gmm.generate_data(300, 11)
    h = gmm.default_hyper(y)
    s = gmm.make_sampler(n, data=y, T=T, seed=5)
    s.initialize()
    s.iterate(T)
    hist = s.history()
    ref = O.gmm_run(n, 5, "stratified", 0.5, y, h, T, 2.0)
    assert np.array_equal(hist["resampled"], ref[:, 1])
    np.testing.assert_allclose(hist["path.grid"], ref[:, 5], rtol=1e-15)
    np.testing.assert_allclose(hist["ess_over_n"], ref[:, 0], rtol=1e-6)
    for k, col in ((1, 2), (2, 3), (3, 4)):
        assert np.all(np.abs(hist[f"accept.{k}"] - ref[:, col]) <= 2), k
    np.testing.assert_allclose(hist["path.integrand"], ref[:, 6], rtol=1e-6)
    assert abs(s.log_zconst - ref[-1, 7]) <= 1e-6 * abs(ref[-1, 7])


def test_conjugate_oracle_acceptance_4():
    """single Normal likelihood of known variance, Normal prior on mu: DS and PS
    within 0.2 of the analytic log evidence (N = 8192, T = 100, prior annealing); mean |error|
    over 20 seeds < 0.05."""
    from paper_1306_5583_b200 import gmm
    from paper_1306_5583_b200.rng import RngStreamSet
    st = RngStreamSet(1, 2024).stream(0)
    lam0 = 1.0
    y = (1.0 + st.normal(0.0, 1.0, 100) / math.sqrt(lam0)).cpu().numpy()
    xi, kappa = 0.0, 0.04
    truth = gmm.conjugate_log_evidence(y, xi, kappa, lam0)
    h = [xi, kappa, 2.0, 1.0, 1.0, lam0]
    err_ds, err_ps = [], []
    for seed in range(20):
        s = gmm.make_sampler(8192, data=y, T=100, seed=100 + seed, hyper=h, components=1)
        s.initialize()
        s.iterate(100)
        d, p = s.log_zconst - truth, s.path_log_zconst() - truth
        assert abs(d) < 0.2 and abs(p) < 0.2, (seed, d, p)
        err_ds.append(d)
        err_ps.append(p)
    assert np.mean(np.abs(err_ds)) < 0.05 and np.mean(np.abs(err_ps)) < 0.05, (err_ds, err_ps)


def test_ds_ps_agreement_acceptance_5():
    """|DS - PS| < 1 over 10 seeds and sd(DS) < 1 (N = 8192, T = 100, 4 components)."""
    from paper_1306_5583_b200 import gmm
    y = gmm.generate_data(100, 1306)
    ds = []
    for seed in range(10):
        s = gmm.make_sampler(8192, data=y, T=100, seed=seed)
        s.initialize()
        s.iterate(100)
        d, p = s.log_zconst, s.path_log_zconst()
        assert abs(d - p) < 1.0, (seed, d, p)
        ds.append(d)
    assert np.std(ds) < 1.0
