"""CPU oracle pinned against the reference (golden draws from rng.py) and SPEC.md's examples.

No GPU: this is the -m "not gpu" suite that makes the oracle trustworthy
before the device kernels are compared with it.
"""

import math
from bisect import bisect_right

import numpy as np
import pytest

from oracle import oracle as O


# ------------------------------------------------------------------ rng.py --
def test_philox_kat(golden):
    for b in golden["philox"]:
        assert O.philox(b["ctr"], b["key"]) == b["out"]


def test_random123_vectors():
    # Random123 philox4x32_10 known-answer vectors
    assert O.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_stream_sequences_bit_exact(golden):
    for s in golden["streams"]:
        st = O.Streams(s["size"], int(s["seed"]))
        i = s["index"]
        for kind, shape, val, ctr in s["ops"]:
            v = st.u01(i) if kind == "u01" else st.normal(i) if kind == "normal" else st.gamma(i, shape)
            assert v.hex() == val, (s["seed"], i, kind, shape)
            assert int(st.counters[i]) == ctr


def test_fills_and_stream_sets_bit_exact(golden):
    for f in golden["fills"]:
        st = O.Streams(4, f["seed"])
        v = st.fill(f["kind"], 3, f["n"], f["shape"] or 1.0)
        assert [x.hex() for x in v] == f["values"]
        assert int(st.counters[3]) == f["counter"]
    for d in golden["draw_sets"]:
        st = O.Streams(d["size"], d["seed"])
        kind = {"u01": "u01", "normal": "normal", "gamma2": "gamma", "gamma05": "gamma"}[d["kind"]]
        shape = {"gamma2": 2.0, "gamma05": 0.5}.get(d["kind"], 1.0)
        v = st.draw_streams(kind, 0, d["size"], shape, nthreads=4)  # thread-count independent
        assert [x.hex() for x in v] == d["values"]
        assert [int(c) for c in st.counters] == d["counters"]


def test_appendix_c_draws():
    st = O.Streams(5, 1306)
    assert st.u01(0) == 0.5012595422834993 and st.u01(0) == 0.9015570423449109
    st = O.Streams(1, 0)
    assert [st.u01(0) for _ in range(2)] == [0.39904647231489565, 0.9722412032044762]


# --------------------------------------------------------------- weights ----
def _ws(values, mode=O.W_SET_LOG):
    v = np.asarray(values, np.float64)
    lw, w = np.empty_like(v), np.empty_like(v)
    ess = O.weights_update(mode, lw, w, v)
    return lw, w, ess


def test_weights_spec_examples():
    lw, w = np.empty(4), np.empty(4)
    assert O.weights_update(O.W_EQUAL, lw, w) == 4 and np.all(w == 0.25)
    lw, w, _ = _ws([0, 0, 0])
    assert np.allclose(w, 1 / 3, atol=1e-15)
    for c in (-7.5, 0.0, 123.0):
        lw, w, _ = _ws([c, c + math.log(2)])
        assert np.allclose(w, [1 / 3, 2 / 3], atol=1e-15)
    lw, w, _ = _ws([1000, 1000])
    assert np.allclose(w, [0.5, 0.5], atol=0)
    lw, w, _ = _ws([0, 0])
    assert np.allclose(lw, -math.log(2), atol=1e-15)
    # add_log_weight
    lw, w, _ = _ws(np.log([0.5, 0.5]))
    O.weights_update(O.W_ADD_LOG, lw, w, np.array([math.log(3), 0.0]))
    assert np.allclose(w, [0.75, 0.25], atol=1e-15)
    lw, w, _ = _ws([0.0, -np.inf])
    O.weights_update(O.W_ADD_LOG, lw, w, np.array([0.0, 5.0]))
    assert list(w) == [1.0, 0.0]
    # linear domain
    lw, w, _ = _ws([2, 2, 2, 2], O.W_SET_LIN)
    assert np.all(w == 0.25)
    O.weights_update(O.W_MUL_LIN, lw, w, np.array([1, 1, 1, 3.0]))
    assert np.allclose(w, [1 / 6, 1 / 6, 1 / 6, 1 / 2], atol=1e-15)
    # ESS
    assert abs(_ws(np.log([0.25] * 4))[2] - 4) < 1e-12
    assert abs(_ws([0.0, -np.inf, -np.inf, -np.inf])[2] - 1) < 1e-12
    assert abs(_ws(np.log([0.5, 0.25, 0.25]))[2] - 8 / 3) < 1e-12


def test_weights_failures():
    with pytest.raises(O.OracleError):
        _ws([-np.inf, -np.inf])
    with pytest.raises(O.OracleError):
        _ws([0.0, np.nan])
    with pytest.raises(O.OracleError):
        _ws([0.0, 0.0], O.W_SET_LIN)


def test_nc_increment_examples():
    assert abs(O.nc_increment(np.log([0.5, 0.5]), np.log([2.0, 4.0])) - math.log(3)) < 1e-15
    lw = np.log(np.array([0.1, 0.2, 0.7]))
    assert abs(O.nc_increment(lw, np.full(3, 1.7)) - 1.7) < 1e-15


# ----------------------------------------------- resampling: exact contract --
def exact_counts(scheme, w, u, m_out=None):
    """Independent pure-Python (arbitrary precision) statement of DESIGN.md's contract."""
    n = len(w)
    m_out = n if m_out is None else m_out
    q = [int(float(x) * 2.0 ** 63) for x in w]
    counts = [0] * n
    if n == 1:
        return [m_out], 0
    base = [0] * n
    if scheme in ("residual", "residual_stratified", "residual_systematic"):
        L = (n - 1).bit_length()
        xs = [float(m_out) * float(x) for x in w]
        base = [int(math.floor(x)) for x in xs]
        q = [int((x - math.floor(x)) * 2.0 ** (63 - L)) for x in xs]
        M = m_out - sum(base)
    else:
        M = m_out
    T = sum(q)
    Q = np.cumsum(np.array(q, dtype=object)).tolist()
    m = [int(x * 2.0 ** 53) for x in u]
    if scheme in ("multinomial", "residual"):
        pos = [(m[k] * T) >> 53 for k in range(M)]
        draws = M
    elif scheme in ("stratified", "residual_stratified"):
        pos = [((k * 2 ** 53 + m[k]) * T) // (M * 2 ** 53) for k in range(M)]
        draws = M
    else:
        pos = [((k * 2 ** 53 + m[0]) * T) // (M * 2 ** 53) for k in range(M)] if M else []
        draws = 1 if M else 0
    for p in pos:
        counts[bisect_right(Q, p)] += 1
    return [b + c for b, c in zip(base, counts)], draws


SCHEMES = list(O.SCHEMES)


def _weights(rng, n, kind):
    if kind == "uniform":
        lw = rng.uniform(-1e-3, 1e-3, n)
    elif kind == "skewed":
        lw = rng.normal(0, 3, n)
    elif kind == "sparse":
        lw = np.where(rng.random(n) < 0.1, rng.normal(0, 1, n), -np.inf)
        lw[rng.integers(n)] = 0.0
    else:  # degenerate
        lw = np.full(n, -50.0)
        lw[0] = 0.0
    return O.normalize_log(lw)[1]


@pytest.mark.parametrize("scheme", SCHEMES)
def test_oracle_matches_exact_contract(scheme):
    rng = np.random.default_rng(1306)
    for trial in range(60):
        n = int(rng.integers(1, 40))
        w = _weights(rng, n, ["uniform", "skewed", "sparse", "degenerate"][trial % 4])
        u = rng.random(n + 1)
        if trial % 7 == 0:
            u[0] = 1 - 2.0 ** -53
        ref, draws = exact_counts(scheme, w, u)
        got, gd = O.resample_counts(scheme, w, u=u)
        assert list(got) == ref and gd == draws, (scheme, n, trial)
        assert got.sum() == n


def test_resample_spec_examples():
    for s in SCHEMES:
        c, _ = O.resample_counts(s, [1.0, 0.0, 0.0], u=[0.5, 0.5, 0.5])
        assert list(c) == [3, 0, 0]
    c, d = O.resample_counts("systematic", [0.5, 0.5], u=[0.3])
    assert list(c) == [1, 1] and d == 1
    c, d = O.resample_counts("residual", [0.5, 0.3, 0.2], u=[], m_out=10)
    assert list(c) == [5, 3, 2] and d == 0  # SPEC.md:162 (pins fl(N W))
    assert list(O.replication_to_parents([2, 0, 1])) == [0, 0, 2]
    assert list(O.replication_to_parents([1] * 7)) == list(range(7))
    assert list(O.replication_to_parents([0, 3, 0])) == [1, 1, 1]
    with pytest.raises(O.OracleError):
        O.replication_to_parents([2, 2, 0])


@pytest.mark.parametrize("n", [1, 2, 3, 49, 98, 103, 1000, 4099])
def test_equal_weights_all_ones(n):
    w = np.full(n, 1.0 / n)
    # plain Residual keeps SPEC.md:162's fl(N W) floors; those are inexact when
    # fl(N * fl(1/N)) < 1 (N = 49, 98, 103, ...: SURVEY F6), and then its
    # R = N leftovers are drawn multinomially -- all-ones is not guaranteed.
    floors_exact = math.floor(float(n) * (1.0 / n)) == 1
    for s in ("stratified", "systematic", "residual", "residual_stratified", "residual_systematic"):
        for u0 in (0.0, 0.5, 1 - 2.0 ** -53):
            c, _ = O.resample_counts(s, w, u=np.full(n, u0))
            assert c.sum() == n
            if s != "residual" or floors_exact:
                assert np.all(c == 1), (s, n, u0)


def test_copy_rows_examples():
    x = np.array([[1.0], [2.0], [3.0]])
    assert O.copy_rows(x.copy(), [0, 1, 2]).ravel().tolist() == [1, 2, 3]
    assert O.copy_rows(x.copy(), [0, 0, 2]).ravel().tolist() == [1, 1, 3]
    assert O.copy_rows(np.array([[1.0], [2.0]]), [1, 0]).ravel().tolist() == [2, 1]  # simultaneity


def test_resample_unnormalized_rejected():
    with pytest.raises(O.OracleError):
        O.resample_counts("stratified", [0.5, 0.6], u=[0.1, 0.2])
    with pytest.raises(O.OracleError):
        O.resample_counts("stratified", [0.5, np.nan], u=[0.1, 0.2])


def test_unbiasedness_acceptance_1():
    """W=(.05,.15,.3,.5), N=4, 4 standard errors."""
    W = np.array([0.05, 0.15, 0.3, 0.5])
    reps = 40000
    st = O.Streams(5, 2024)
    for s in SCHEMES:
        acc = np.zeros((reps, 4))
        for r in range(reps):
            acc[r] = O.resample_counts(s, W, streams=st, stream=4)[0]
        mean, sd = acc.mean(0), acc.std(0) + 1e-12
        assert np.all(np.abs(mean - 4 * W) <= 4 * sd / math.sqrt(reps) + 1e-12), (s, mean)


def test_draw_counts_pinned():
    st = O.Streams(9, 5)
    w = O.normalize_log(np.random.default_rng(0).normal(size=8))[1]
    for s, expect in [("multinomial", 8), ("stratified", 8), ("systematic", 1)]:
        c0 = int(st.counters[8])
        _, d = O.resample_counts(s, w, streams=st, stream=8)
        assert d == expect and int(st.counters[8]) - c0 == expect


# -------------------------------------------------------------------- pf -----
def test_cv_llh_examples():
    assert O.cv_llh(0, 0, 0, 0) == 0.0
    assert abs(O.cv_llh(0.1, 0, 0, 0) - (-5.5 * math.log(1.1))) < 1e-15
    # SPEC.md:471 prints "~ -0.524180"; -5.5 ln 1.1 is -0.5242060 (the decimal is a typo, the
    # symbolic value is what the formula gives)
    assert abs(O.cv_llh(0.1, 0, 0, 0) + 0.5242060) < 1e-7
    assert O.cv_llh(0.3, -0.2, 0.1, 0.1) == O.cv_llh(-0.1, 0.4, 0.1, 0.1)


def test_pf_run_properties():
    obs = np.cumsum(np.random.default_rng(3).normal(0, 0.1, (50, 2)), axis=0)
    h1 = O.pf_run(1000, 7, "systematic", 0.5, obs, nthreads=1)
    h4 = O.pf_run(1000, 7, "systematic", 0.5, obs, nthreads=4)
    assert np.array_equal(h1, h4)  # backend equivalence
    assert np.all((h1[:, 1] == 1) == (h1[:, 0] < 0.5))  # history invariant
    assert np.all(h1[:, 0] <= 1 + 1e-12) and np.all(h1[:, 0] > 0)
