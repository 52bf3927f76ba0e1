"""The paper's Gaussian-mixture SMC sampler on the device (mirror of smckit
example-gmm; BASELINE config 3).

Tempered targets pi_alpha(theta) ∝ prior(theta) lik(theta)^alpha with a
prior-annealing schedule alpha_t = (t/T)^p; each iteration re-weights by
(alpha_t - alpha_{t-1}) llh (accumulating the direct log Z estimate), resamples
when ESS/N < threshold, then applies the three random-walk Metropolis blocks
(mu, log lambda, logit omega).  The path-sampling integrand is llh (grid alpha),
so log Z_PS is the trapezoid rule over the history.

    s = gmm.make_sampler(1 << 20, seed=1306)      # 1000 synthetic points, T = 100
    s.initialize(); s.iterate(100)
    ds, ps = s.log_zconst, s.path_log_zconst()
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _abi
from .core import ROW_MAJOR, Sampler, StateMatrix
from .exec import ParticleKernelOp, PathEval
from .resample import ResampleScheme
from .rng import RngStreamSet

__all__ = ["GmmState", "generate_data", "default_hyper", "alpha_linear", "alpha_prior", "gmm_init", "gmm_move_smc",
           "gmm_move_mu", "gmm_move_lambda", "gmm_move_weight", "gmm_path", "make_sampler", "ROW", "R",
           "TRUE_MU", "TRUE_LAMBDA", "TRUE_OMEGA", "MAX_R", "conjugate_log_evidence"]

R = 4     # the paper's 4-component model (config 3); 1 <= components <= MAX_R
MAX_R = 4
ROW = 16  # SMC_GMM_ROW: mu[4] lambda[4] omega[4] log_prior log_likelihood pad pad
TRUE_MU = (-3.0, 0.0, 3.0, 6.0)
TRUE_LAMBDA = 2.0
TRUE_OMEGA = 0.25


def generate_data(n=1000, seed=1306, device="cuda"):
    """n draws from the 4-component truth: u -> component floor(4u),
    then mu_c + z / sqrt(lambda), all from stream 0 of RngStreamSet(1, seed)."""
    st = RngStreamSet(1, seed, device).stream(0)
    u = st.uniform01(n).cpu().numpy()
    z = st.normal(0.0, 1.0, n).cpu().numpy()
    c = np.minimum((u * R).astype(np.int64), R - 1)
    return np.asarray(TRUE_MU)[c] + z / math.sqrt(TRUE_LAMBDA)


def default_hyper(data, lambda_known=0.0):
    """xi = midrange, kappa = 1/R^2, nu = 2, chi = 50/R^2, rho = 1 (R = data range);
    6th value lambda_known (0: lambda unknown with the Gamma prior)."""
    lo, hi = float(np.min(data)), float(np.max(data))
    rng = hi - lo
    return [0.5 * (lo + hi), 1.0 / (rng * rng), 2.0, 50.0 / (rng * rng), 1.0, float(lambda_known)]


def conjugate_log_evidence(data, xi, kappa, lam):
    """Closed-form log p(y) for y_k ~ N(mu, 1/lam), mu ~ N(xi, 1/kappa) (the conjugate oracle,
    SPEC.md:586-587): y ~ N(xi 1, I/lam + 11'/kappa)."""
    y = np.asarray(data, np.float64) - xi
    n = y.size
    s2, t2 = 1.0 / lam, 1.0 / kappa
    logdet = (n - 1) * math.log(s2) + math.log(s2 + n * t2)
    quad = (float(np.dot(y, y)) - t2 * float(y.sum()) ** 2 / (s2 + n * t2)) / s2
    return -0.5 * n * math.log(2 * math.pi) - 0.5 * logdet - 0.5 * quad


def alpha_linear(T):
    """alpha(t) = t / T."""
    return lambda t: t / T


def alpha_prior(T, p=2.0):
    """alpha(t) = (t / T)^p (p = 2 by default)."""
    return lambda t: (t / T) ** p


class GmmState(StateMatrix):
    """StateMatrix<RowMajor, 16, double> + data, hyperparameters, alpha."""

    def __init__(self, size, device="cuda", components=R):
        super().__init__(size, ROW, ROW_MAJOR, device)
        if not 1 <= int(components) <= MAX_R:
            raise ValueError(f"components must be in [1, {MAX_R}]")
        self.r = int(components)
        self.y = None
        self.hyper = None
        self._hyper_c = None
        self.alpha = 0.0
        self.alpha_inc = 0.0
        self.sds = (0.0, 0.0, 0.0)

    def set_data(self, data, hyper=None):
        arr = np.ascontiguousarray(data, dtype=np.float64).ravel()
        if not 0 < arr.size <= 4096:
            raise ValueError("GMM data must hold 1..4096 points")
        self.y = torch.as_tensor(arr).to(self.device)
        h = list(default_hyper(arr) if hyper is None else hyper)
        h += [0.0] * (6 - len(h))
        if len(h) != 6:
            raise ValueError("hyper: xi, kappa, nu, chi, rho[, lambda_known]")
        self.hyper = h
        self._hyper_c = (ctypes.c_double * 6)(*self.hyper)

    @property
    def lambda_known(self):
        return self.hyper is not None and self.hyper[5] > 0

    def set_alpha(self, a):
        """gmm_state::alpha: clamp to [0, 1], track the increment."""
        a = min(max(a, 0.0), 1.0)
        if a == 0.0:
            self.alpha_inc, self.alpha = 0.0, 0.0
        else:
            self.alpha_inc, self.alpha = a - self.alpha, a


def _ws(system, n):
    ws = getattr(system, "_gmm_ws", None)
    if ws is None:
        ws = system._gmm_ws = _abi.Workspace(system.device)
    return ws.get(_abi.lib().smc_gmm_workspace_bytes(n))


def gmm_init(system, param=None):
    """gmm_init: data (param) if given, prior draws, alpha = 0, NC reset."""
    v = system.value
    if param is not None:
        if isinstance(param, dict):
            v.set_data(param["data"], param.get("hyper"))
        else:
            v.set_data(param)
    if v.y is None:
        raise RuntimeError("gmm_init: no data")
    v.set_alpha(0.0)
    v.pending = None
    system.weight_set.reset_log_zconst()
    _abi.call("smc_gmm_init", _abi.ptr(v.raw), system.size, v.r, system.stream_base, system.rng_set.seed,
              _abi.ptr(system.rng_set.counters), _abi.ptr(v.y), v.y.numel(), v._hyper_c, _abi.stream())
    return None


def gmm_move_smc(schedule):
    """gmm_move_smc: alpha_t, proposal scales, incw = dalpha llh,
    nc.add_log_weight + add_log_weight (one fused kernel)."""

    def kernel(iter_, system):
        v = system.value
        v.set_alpha(schedule(iter_))
        a = max(v.alpha, 0.02)
        v.sds = (0.15 / a, (1 + math.sqrt(1 / a)) * 0.15, (1 + math.sqrt(1 / a)) * 0.2)
        w = system.weight_set
        ws, nb = _ws(system, system.size)
        _abi.call("smc_gmm_reweight", _abi.ptr(v.raw), _abi.ptr(w.lw_raw), system.size, v.alpha_inc, w.state_ptr,
                  None, ws, nb, _abi.stream())
        return None

    return ParticleKernelOp(kernel, name="gmm_move_smc")


def _mh(block, name):
    def kernel(iter_, system):
        v = system.value
        acc = torch.zeros(1, dtype=torch.int64, device=system.device)
        _abi.call("smc_gmm_mh", block, _abi.ptr(v.raw), system.size, v.r, system.stream_base, system.rng_set.seed,
                  _abi.ptr(system.rng_set.counters), _abi.ptr(v.y), v.y.numel(), v._hyper_c, v.alpha,
                  v.sds[block], _abi.ptr(acc), _abi.stream())
        return acc  # accepted count

    return ParticleKernelOp(kernel, name=name)


def gmm_move_mu():
    return _mh(0, "gmm_move_mu")


def gmm_move_lambda():
    return _mh(1, "gmm_move_lambda")


def gmm_move_weight():
    return _mh(2, "gmm_move_weight")


def gmm_path():
    """gmm_path: integrand = log-likelihood, grid = alpha."""
    return PathEval(lambda it, system: (system.value.alpha, system.value.data.view(-1)[13:], ROW))


def make_sampler(n, data=None, T=100, power=2.0, scheme=ResampleScheme.Stratified, threshold=0.5, seed=0,
                 hyper=None, components=R, device="cuda"):
    """The paper's GMM main: init, move_smc, mu/lambda/weight MCMC, path sampling.

    components: r (1..4).  hyper[5] = lambda_known > 0 gives the conjugate-oracle model (lambda
    fixed, no lambda block); r = 1 has no weight block (omega = 1)."""
    v = GmmState(n, device, components)
    v.set_data(generate_data(1000, 1306, device) if data is None else data, hyper)
    s = Sampler(n, scheme, threshold, seed, value=v, device=device)
    s.set_init(gmm_init)
    s.add_move(gmm_move_smc(alpha_prior(T, power) if power != 1 else alpha_linear(T)), False)
    s.add_mcmc(gmm_move_mu(), False)
    if not v.lambda_known:
        s.add_mcmc(gmm_move_lambda(), True)
    if v.r > 1:
        s.add_mcmc(gmm_move_weight(), True)
    s.set_path(gmm_path())
    return s
