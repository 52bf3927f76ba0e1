"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE -- the checker).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_1306_5583_b200) never does; it has no CPU path.

Every function cites the reference line it restates (see smc_oracle.c).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libsmc_oracle.so")
_lib = None

MULTINOMIAL, RESIDUAL, STRATIFIED, SYSTEMATIC, RESIDUAL_STRATIFIED, RESIDUAL_SYSTEMATIC = range(6)
SCHEMES = {
    "multinomial": MULTINOMIAL, "residual": RESIDUAL, "stratified": STRATIFIED,
    "systematic": SYSTEMATIC, "residual_stratified": RESIDUAL_STRATIFIED,
    "residual_systematic": RESIDUAL_SYSTEMATIC,
}
W_SET_LOG, W_ADD_LOG, W_SET_LIN, W_MUL_LIN, W_EQUAL = range(5)

_P = np.ctypeslib.ndpointer
_f64 = _P(dtype=np.float64, flags="C_CONTIGUOUS")
_u64 = _P(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32 = _P(dtype=np.int32, flags="C_CONTIGUOUS")
_u32 = _P(dtype=np.uint32, flags="C_CONTIGUOUS")


def build():
    """Compile oracle/smc_oracle.c (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "smc_oracle.c"))):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_philox4x32_10.argtypes = [_u32, C.c_uint32, C.c_uint32, _u32]
        L.orc_u01.restype = C.c_double
        L.orc_u01.argtypes = [_u64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_std_normal.restype = C.c_double
        L.orc_std_normal.argtypes = [_u64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_std_gamma.restype = C.c_double
        L.orc_std_gamma.argtypes = [_u64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double]
        L.orc_fill.argtypes = [C.c_int, _u64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, _f64,
                               C.c_int64]
        L.orc_draw_streams.argtypes = [C.c_int, _u64, C.c_uint64, C.c_int64, C.c_uint32, C.c_uint32,
                                       C.c_double, _f64, C.c_int]
        L.orc_weights_update.argtypes = [C.c_int, _f64, _f64, C.c_void_p, C.c_int64,
                                         C.POINTER(C.c_double)]
        L.orc_nc_increment.restype = C.c_double
        L.orc_nc_increment.argtypes = [_f64, _f64, C.c_int64]
        L.orc_resample_counts.argtypes = [C.c_int, _f64, C.c_int64, C.c_int64, _u64, C.c_uint64, C.c_uint32,
                                          C.c_uint32, C.c_void_p, C.c_int64, _i32,
                                          C.POINTER(C.c_int64)]
        L.orc_replication_to_parents.argtypes = [_i32, C.c_int64, _i32]
        L.orc_copy_rows.argtypes = [_f64, C.c_int64, C.c_int64, _i32]
        L.orc_cv_llh.restype = C.c_double
        L.orc_cv_llh.argtypes = [C.c_double] * 4
        L.orc_cv_init.argtypes = [_f64, C.c_int64, _u64, C.c_uint32, C.c_uint32, _f64, _f64, C.c_int]
        L.orc_cv_move.argtypes = [_f64, C.c_int64, _u64, C.c_uint32, C.c_uint32, _f64, _f64, C.c_int]
        L.orc_weighted_sum.argtypes = [_f64, _f64, C.c_int64, C.c_int64, _f64]
        L.orc_pf_run.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_double, _f64, C.c_int64, _f64,
                                 C.c_void_p, C.c_void_p, C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _key(seed):
    seed = int(seed) % (1 << 64)
    return seed & 0xFFFFFFFF, seed >> 32


# ---------------------------------------------------------------- rng.py ----
def philox(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(np.asarray(ctr, np.uint32), int(key[0]), int(key[1]), out)
    return [int(v) for v in out]


class Streams:
    """N+1 counter streams (rng.py:138-170) with the oracle's draw functions."""

    def __init__(self, size, seed=0):
        self.size = int(size)
        self.seed = int(seed) % (1 << 64)
        self.k0, self.k1 = _key(self.seed)
        self.counters = np.zeros(self.size, np.uint64)

    def u01(self, i):
        return lib().orc_u01(self.counters, i, self.k0, self.k1)

    def normal(self, i):
        return lib().orc_std_normal(self.counters, i, self.k0, self.k1)

    def gamma(self, i, shape):
        return lib().orc_std_gamma(self.counters, i, self.k0, self.k1, shape)

    def fill(self, kind, i, n, shape=1.0):
        out = np.empty(int(n), np.float64)
        lib().orc_fill({"u01": 0, "normal": 1, "gamma": 2}[kind], self.counters, i, self.k0, self.k1,
                       float(shape), out, int(n))
        return out

    def draw_streams(self, kind, first, n, shape=1.0, nthreads=1):
        out = np.empty(int(n), np.float64)
        lib().orc_draw_streams({"u01": 0, "normal": 1, "gamma": 2}[kind], self.counters, first, int(n),
                               self.k0, self.k1, float(shape), out, int(nthreads))
        return out


# --------------------------------------------------------------- weights ----
def weights_update(mode, lw, w, values=None):
    """In-place update of normalized (lw, w); returns ESS."""
    ess = C.c_double()
    vp = None if values is None else np.ascontiguousarray(values, np.float64).ctypes.data
    keep = values
    rc = lib().orc_weights_update(mode, lw, w, vp, lw.size, C.byref(ess))
    del keep
    if rc:
        raise OracleError(f"weights_update rc={rc}")
    return ess.value


def normalize_log(values):
    v = np.ascontiguousarray(values, np.float64)
    lw = np.empty_like(v)
    w = np.empty_like(v)
    ess = weights_update(W_SET_LOG, lw, w, v)
    return lw, w, ess


def nc_increment(lw, incw):
    return lib().orc_nc_increment(np.ascontiguousarray(lw, np.float64),
                                  np.ascontiguousarray(incw, np.float64), len(lw))


# -------------------------------------------------------------- resample ----
def resample_counts(scheme, w, u=None, streams=None, stream=None, m_out=None):
    """Replication counts under the pinned integer contract.  Returns (counts, draws)."""
    if isinstance(scheme, str):
        scheme = SCHEMES[scheme]
    w = np.ascontiguousarray(w, np.float64)
    n = w.size
    m_out = n if m_out is None else int(m_out)
    counts = np.zeros(n, np.int32)
    draws = C.c_int64()
    if u is not None:
        u = np.ascontiguousarray(u, np.float64)
        ctrs = np.zeros(1, np.uint64)
        rc = lib().orc_resample_counts(scheme, w, n, m_out, ctrs, 0, 0, 0, u.ctypes.data, u.size, counts,
                                       C.byref(draws))
    else:
        rc = lib().orc_resample_counts(scheme, w, n, m_out, streams.counters, stream, streams.k0, streams.k1,
                                       None, 0, counts, C.byref(draws))
    if rc:
        raise OracleError(f"resample rc={rc}")
    return counts, draws.value


def replication_to_parents(counts):
    counts = np.ascontiguousarray(counts, np.int32)
    parents = np.empty(counts.size, np.int32)
    rc = lib().orc_replication_to_parents(counts, counts.size, parents)
    if rc:
        raise OracleError("count sum mismatch")
    return parents


def copy_rows(x, parents):
    x = np.ascontiguousarray(x, np.float64)
    n, d = x.shape
    lib().orc_copy_rows(x, n, d, np.ascontiguousarray(parents, np.int32))
    return x


# ------------------------------------------------------------------- pf -----
def cv_llh(xp, yp, xo, yo):
    return lib().orc_cv_llh(xp, yp, xo, yo)


def cv_init(n, streams, obs0, nthreads=1):
    x = np.empty((n, 4), np.float64)
    llh = np.empty(n, np.float64)
    lib().orc_cv_init(x, n, streams.counters, streams.k0, streams.k1,
                      np.ascontiguousarray(obs0, np.float64), llh, nthreads)
    return x, llh


def cv_move(x, streams, obs_t, nthreads=1):
    incw = np.empty(x.shape[0], np.float64)
    lib().orc_cv_move(x, x.shape[0], streams.counters, streams.k0, streams.k1,
                      np.ascontiguousarray(obs_t, np.float64), incw, nthreads)
    return incw


def pf_run(n, seed, scheme, threshold, obs, nthreads=1, want_state=False):
    """Full PF run; returns hist (T x 5: ess_over_n, resampled, pos.0, pos.1, log_zconst)."""
    if isinstance(scheme, str):
        scheme = SCHEMES[scheme]
    obs = np.ascontiguousarray(obs, np.float64)
    T = obs.shape[0]
    hist = np.zeros((T, 5), np.float64)
    x = np.empty((n, 4), np.float64) if want_state else None
    lw = np.empty(n, np.float64) if want_state else None
    rc = lib().orc_pf_run(n, seed, scheme, threshold, obs, T, hist,
                          None if x is None else x.ctypes.data, None if lw is None else lw.ctypes.data,
                          nthreads)
    if rc:
        raise OracleError(f"pf_run rc={rc}")
    return (hist, x, lw) if want_state else hist


# ------------------------------------------------------------------ gmm -----
def _gmm_sigs():
    L = lib()
    if getattr(L, "_gmm_ok", False):
        return L
    L.orc_gmm_llh.restype = C.c_double
    L.orc_gmm_llh.argtypes = [_f64, C.c_int, _f64, C.c_int]
    L.orc_gmm_lprior.restype = C.c_double
    L.orc_gmm_lprior.argtypes = [_f64, C.c_int, _f64]
    L.orc_gmm_init.argtypes = [_f64, C.c_int64, C.c_int, _u64, C.c_uint32, C.c_uint32, _f64, C.c_int, _f64, C.c_int]
    L.orc_gmm_mh.restype = C.c_int64
    L.orc_gmm_mh.argtypes = [C.c_int, _f64, C.c_int64, C.c_int, _u64, C.c_uint32, C.c_uint32, _f64, C.c_int, _f64,
                             C.c_double, C.c_double, C.c_int]
    L.orc_gmm_run.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_double, _f64, C.c_int, _f64, C.c_int,
                              C.c_double, _f64, C.c_int]
    L.orc_gmm_run_steps.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_double, _f64, C.c_int, _f64,
                                    C.c_int, C.c_int, C.c_double, _f64, C.c_int]
    L._gmm_ok = True
    return L


def _h6(h):
    h = list(h) + [0.0] * (6 - len(h))
    return np.ascontiguousarray(h[:6], np.float64)


def gmm_llh(row, y, r=4):
    return _gmm_sigs().orc_gmm_llh(np.ascontiguousarray(row, np.float64), r, np.ascontiguousarray(y, np.float64),
                                   len(y))


def gmm_lprior(row, h, r=4):
    return _gmm_sigs().orc_gmm_lprior(np.ascontiguousarray(row, np.float64), r, _h6(h))


def gmm_init(n, streams, y, h, r=4, nthreads=1):
    x = np.zeros((n, 16), np.float64)
    y = np.ascontiguousarray(y, np.float64)
    _gmm_sigs().orc_gmm_init(x, n, r, streams.counters, streams.k0, streams.k1, y, len(y), _h6(h), nthreads)
    return x


def gmm_mh(block, x, streams, y, h, alpha, sd, r=4, nthreads=1):
    y = np.ascontiguousarray(y, np.float64)
    return _gmm_sigs().orc_gmm_mh(block, x, x.shape[0], r, streams.counters, streams.k0, streams.k1, y, len(y),
                                  _h6(h), alpha, sd, nthreads)


def gmm_run(n, seed, scheme, threshold, y, h, T, power, r=4, nthreads=1, steps=None):
    """hist (steps+1) x 8: ess_over_n resampled acc_mu acc_lambda acc_weight alpha U_t log_zconst.
    steps < T: only the first `steps` iterations of the T-iteration schedule."""
    if isinstance(scheme, str):
        scheme = SCHEMES[scheme]
    y = np.ascontiguousarray(y, np.float64)
    steps = T if steps is None else int(steps)
    hist = np.zeros((steps + 1, 8), np.float64)
    rc = _gmm_sigs().orc_gmm_run_steps(n, r, seed, scheme, threshold, y, len(y), _h6(h), T, steps, power, hist,
                                       nthreads)
    if rc:
        raise OracleError(f"gmm_run rc={rc}")
    return hist
