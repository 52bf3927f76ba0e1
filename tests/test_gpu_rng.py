"""Device Philox streams vs the reference's own draws (tests/golden/rng_golden.json)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def ulps(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    sp = np.spacing(np.maximum(np.abs(a), np.abs(b)))
    return np.max(np.abs(a - b) / sp) if a.size else 0.0


def test_philox_blocks_kat(golden):
    from paper_1306_5583_b200 import _abi
    for b in golden["philox"]:
        seed = b["key"][0] | (b["key"][1] << 32)
        ctr = torch.tensor(np.array(b["ctr"], np.uint32).view(np.int32)).cuda()
        out = torch.zeros(4, dtype=torch.int32, device="cuda")
        _abi.call("smc_philox_blocks", _abi.ptr(ctr), 1, seed, _abi.ptr(out), _abi.stream())
        got = out.cpu().numpy().view(np.uint32).tolist()
        assert got == b["out"]


def test_streams_match_reference(golden):
    from paper_1306_5583_b200 import RngStreamSet
    worst = 0.0
    for s in golden["streams"]:
        if s["size"] > 4096:
            continue
        ss = RngStreamSet(s["size"], int(s["seed"]))
        st = ss.stream(s["index"])
        for kind, shape, val, ctr in s["ops"]:
            ref = float.fromhex(val)
            if kind == "u01":
                assert st.uniform01() == ref  # bit-exact
            elif kind == "normal":
                v = st.normal()
                worst = max(worst, ulps(v, ref))
            else:
                v = st.gamma(shape)
                assert abs(v - ref) <= 1e-12 * abs(ref)
            assert ss.counters_host()[s["index"]] == ctr
    assert worst <= 8, worst


def test_fill_matches_reference(golden):
    from paper_1306_5583_b200 import RngStreamSet
    for f in golden["fills"]:
        ss = RngStreamSet(4, f["seed"])
        st = ss.stream(3)
        ref = np.array([float.fromhex(v) for v in f["values"]])
        if f["kind"] == "u01":
            got = st.uniform01(f["n"]).cpu().numpy()
            assert np.array_equal(got, ref)
        elif f["kind"] == "normal":
            got = st.normal(0.0, 1.0, f["n"]).cpu().numpy()
            assert ulps(got, ref) <= 8
        else:
            got = st.gamma(f["shape"], 1.0, f["n"]).cpu().numpy()
            np.testing.assert_allclose(got, ref, rtol=1e-12)
        assert ss.counters_host()[3] == f["counter"]


def test_per_stream_draws_match_reference(golden):
    from paper_1306_5583_b200 import RngStreamSet
    for d in golden["draw_sets"]:
        ss = RngStreamSet(d["size"], d["seed"])
        kind = {"u01": 0, "normal": 1, "gamma2": 2, "gamma05": 2}[d["kind"]]
        shape = {"gamma2": 2.0, "gamma05": 0.5}.get(d["kind"], 1.0)
        got = ss.draw_streams(kind, 0, d["size"], shape).cpu().numpy()
        ref = np.array([float.fromhex(v) for v in d["values"]])
        if kind == 0:
            assert np.array_equal(got, ref)
        elif kind == 1:
            assert ulps(got, ref) <= 8
        else:
            np.testing.assert_allclose(got, ref, rtol=1e-12)
        assert ss.counters_host() == d["counters"]


def test_moments_and_ranges():
    """SPEC.md:229-231, :235 statistical checks."""
    from scipy import stats

    from paper_1306_5583_b200 import RngStreamSet
    st = RngStreamSet(2, 77).stream(1)
    u = st.uniform01(100000).cpu().numpy()
    assert u.min() >= 0 and u.max() < 1
    z = st.normal(0, 1, 100000).cpu().numpy()
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.03
    g = st.gamma(2.0, 3.0, 20000).cpu().numpy()
    assert abs(g.mean() - 6) < 4 * math.sqrt(18 / 20000)
    assert stats.kstest(u[:10000], "uniform").pvalue > 0.001
    assert stats.kstest(z[:10000], "norm").pvalue > 0.001


def test_stream_errors():
    from paper_1306_5583_b200 import RngStreamSet
    with pytest.raises(ValueError):
        RngStreamSet(0)
    ss = RngStreamSet(3, 1)
    with pytest.raises(IndexError):
        ss.stream(3)
    with pytest.raises(ValueError):
        ss.stream(0).normal(0, -1)
    with pytest.raises(ValueError):
        ss.stream(0).gamma(0.0)
    assert RngStreamSet(2, (1 << 64) + 5).seed == 5


def test_reference_primitives_on_device_counters(golden):
    """smckit's kernel-callable primitives (rng.py:59-135) by name, on device counters."""
    from paper_1306_5583_b200 import (RngStreamSet, fill_std_gamma, fill_std_normal, fill_u01, philox_block,
                                      sample_gamma, sample_normal, sample_uniform01, std_gamma, std_normal, u01)
    for b in golden["philox"]:
        assert list(philox_block(*b["ctr"], *b["key"])) == b["out"]
    for s in golden["streams"]:
        if s["size"] > 4096:
            continue
        ss = RngStreamSet(s["size"], int(s["seed"]))
        k0, k1 = ss.key
        for kind, shape, val, ctr in s["ops"]:
            ref = float.fromhex(val)
            if kind == "u01":
                assert u01(ss.counters, s["index"], k0, k1) == ref
            elif kind == "normal":
                assert ulps(std_normal(ss.counters, s["index"], k0, k1), ref) <= 8
            else:
                assert abs(std_gamma(ss.counters, s["index"], k0, k1, shape) - ref) <= 1e-12 * abs(ref)
            assert ss.counters_host()[s["index"]] == ctr
    for f in golden["fills"]:
        ss = RngStreamSet(4, f["seed"])
        k0, k1 = ss.key
        out = torch.empty(f["n"], dtype=torch.float64, device="cuda")
        ref = np.array([float.fromhex(v) for v in f["values"]])
        if f["kind"] == "u01":
            assert np.array_equal(fill_u01(ss.counters, 3, k0, k1, out).cpu().numpy(), ref)
        elif f["kind"] == "normal":
            assert ulps(fill_std_normal(ss.counters, 3, k0, k1, out).cpu().numpy(), ref) <= 8
        else:
            np.testing.assert_allclose(fill_std_gamma(ss.counters, 3, k0, k1, f["shape"], out).cpu().numpy(), ref,
                                       rtol=1e-12)
        assert ss.counters_host()[3] == f["counter"]
    st = RngStreamSet(2, 5).stream(1)
    assert 0.0 <= sample_uniform01(st) < 1.0 and isinstance(sample_normal(st, 1.0, 2.0), float)
    assert sample_gamma(st, 2.0, 3.0) > 0


def test_nc_add_log_weight_spec_example():
    """W = (0.5, 0.5), incw = (ln 2, ln 4) -> increment ln 3; weights unchanged."""
    from paper_1306_5583_b200 import NormalizingConstant, WeightSet, nc_add_log_weight
    ws = WeightSet(2)
    nc = NormalizingConstant(ws)
    before = ws.read_weight().cpu().numpy()
    nc_add_log_weight(nc, [math.log(2), math.log(4)], ws)
    assert abs(nc.log_zconst - math.log(3)) < 1e-15
    assert np.array_equal(ws.read_weight().cpu().numpy(), before)
    nc_add_log_weight(nc, [0.7, 0.7], ws)  # all equal c -> increment exactly c
    assert abs(nc.log_zconst - (math.log(3) + 0.7)) < 1e-15
