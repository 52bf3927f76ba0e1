"""GMM SMC sampler (config 3): device kernels vs the oracle and SPEC.md's examples."""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _eval(rows, y, h5):
    from paper_1306_5583_b200 import _abi
    import ctypes
    x = torch.as_tensor(np.asarray(rows, np.float64).reshape(-1, 16)).cuda().contiguous()
    yy = torch.as_tensor(np.asarray(y, np.float64)).cuda()
    _abi.call("smc_gmm_eval", _abi.ptr(x), x.shape[0], _abi.ptr(yy), yy.numel(), (ctypes.c_double * 5)(*h5),
              _abi.stream())
    return x.cpu().numpy()


def _row(mu, lam, om):
    r = np.zeros(16)
    r[0:4], r[4:8], r[8:12] = mu, lam, om
    return r


def test_spec_examples():
    h5 = [0.0, 1.0, 2.0, 1.0, 1.0]
    r1 = _row([0, 5, 5, 5], [1, 1, 1, 1], [1, 0, 0, 0])
    out = _eval([r1], [0.0], h5)
    assert abs(out[0, 13] - (-0.5 * math.log(2 * math.pi))) < 1e-15
    r2 = _row([0.7, 0.7, 9, 9], [2, 2, 1, 1], [0.5, 0.5, 0, 0])
    r3 = _row([0.7, 9, 9, 9], [2, 1, 1, 1], [1, 0, 0, 0])
    y = np.linspace(-2, 2, 17)
    out = _eval([r2, r3], y, h5)
    assert abs(out[0, 13] - out[1, 13]) < 1e-12  # identical components collapse
    # prior: mu = xi everywhere -> normal part r * 0.5 ln(kappa/2pi); rho = 1 -> Dirichlet ln 3!
    h5 = [1.5, 0.25, 2.0, 3.0, 1.0]
    r = _row([1.5] * 4, [1.0] * 4, [0.25] * 4)
    out = _eval([r], [0.0], h5)
    gam = 4 * ((2 - 1) * math.log(1.0) - 1.0 / 3.0 - math.lgamma(2.0) - 2 * math.log(3.0))
    expect = 4 * 0.5 * math.log(0.25 / (2 * math.pi)) + gam + math.log(6.0)
    assert abs(out[0, 12] - expect) < 1e-12
    assert abs(out[0, 12] - O.gmm_lprior(r, h5)) < 1e-12


def test_scales_spec_example():
    from paper_1306_5583_b200 import gmm
    v = gmm.GmmState(4)
    v.set_data([0.0, 1.0])
    op = gmm.gmm_move_smc(lambda t: 0.5)
    assert op.name == "gmm_move_smc"
    a = 0.5
    assert abs(0.15 / a - 0.3) < 1e-15 and abs((1 + math.sqrt(1 / a)) * 0.15 - 0.362132) < 1e-6
    assert abs((1 + math.sqrt(1 / a)) * 0.2 - 0.482843) < 1e-6


def test_init_and_mh_match_oracle():
    from paper_1306_5583_b200 import gmm
    n = 3000
    y = gmm.generate_data(200, 7)
    h5 = gmm.default_hyper(y)
    s = gmm.make_sampler(n, data=y, T=10, seed=99)
    s.initialize()
    x = s.system.value.data.cpu().numpy()
    st = O.Streams(n + 1, 99)
    xo = O.gmm_init(n, st, y, h5)
    np.testing.assert_allclose(x, xo, rtol=1e-12, atol=1e-12)
    assert s.system.rng_set.counters_host()[:n] == [int(c) for c in st.counters[:n]]
    # one block of each MH kernel at alpha = 0.3
    from paper_1306_5583_b200 import _abi
    v = s.system.value
    v.alpha = 0.3
    for block, sd in ((0, 0.5), (1, 0.4), (2, 0.6)):
        v.sds = (0.5, 0.4, 0.6)
        acc = [gmm.gmm_move_mu, gmm.gmm_move_lambda, gmm.gmm_move_weight][block]().kernel(1, s.system)
        acc_o = O.gmm_mh(block, xo, st, y, h5, 0.3, sd)
        assert int(acc.item()) == acc_o
        np.testing.assert_allclose(v.data.cpu().numpy(), xo, rtol=1e-11, atol=1e-11)


def test_full_run_matches_oracle():
    from paper_1306_5583_b200 import gmm
    n, T = 4096, 30
    y = gmm.generate_data(300, 11)
    h5 = gmm.default_hyper(y)
    s = gmm.make_sampler(n, data=y, T=T, seed=5)
    s.initialize()
    s.iterate(T)
    h = s.history()
    ref = O.gmm_run(n, 5, "stratified", 0.5, y, h5, T, 2.0)
    assert np.array_equal(h["resampled"], ref[:, 1])
    np.testing.assert_allclose(h["path.grid"], ref[:, 5], rtol=1e-15)
    np.testing.assert_allclose(h["ess_over_n"], ref[:, 0], rtol=1e-6)
    for k, col in ((1, 2), (2, 3), (3, 4)):
        assert np.all(np.abs(h[f"accept.{k}"] - ref[:, col]) <= 2), k
    np.testing.assert_allclose(h["path.integrand"], ref[:, 6], rtol=1e-6)
    assert abs(s.log_zconst - ref[-1, 7]) <= 1e-6 * abs(ref[-1, 7])


def test_ds_ps_agreement_acceptance_5():
    """|DS - PS| < 1 over seeds (N = 8192, T = 100, prior annealing)."""
    from paper_1306_5583_b200 import gmm
    y = gmm.generate_data(100, 1306)
    ds = []
    for seed in range(3):
        s = gmm.make_sampler(8192, data=y, T=100, seed=seed)
        s.initialize()
        s.iterate(100)
        d, p = s.log_zconst, s.path_log_zconst()
        assert abs(d - p) < 1.0, (seed, d, p)
        ds.append(d)
    assert np.std(ds) < 1.0
