"""WeightSet, monitors, NC and the PF kernels vs the oracle (fp64, tolerance 1e-12 / 1e-6 relative)."""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-6  # north_star: log-weights, ESS, monitors, log Z within 1e-6 relative in fp64


def test_weights_spec_examples_device():
    from paper_1306_5583_b200 import WeightSet, _abi
    ws = WeightSet(4)
    assert ws.read_weight().tolist() == [0.25] * 4 and ws.ess() == 4
    ws = WeightSet(3)
    ws.set_log_weight([0.0, 0.0, 0.0])
    assert np.allclose(ws.read_weight().cpu(), 1 / 3, atol=1e-15)
    ws = WeightSet(2)
    ws.set_log_weight([1000.0, 1000.0])
    assert ws.read_weight().tolist() == [0.5, 0.5]
    ws.set_log_weight([5.0, 5.0 + math.log(2)])
    assert np.allclose(ws.read_weight().cpu(), [1 / 3, 2 / 3], atol=1e-15)
    ws.set_log_weight(np.log([0.5, 0.5]))
    ws.add_log_weight([math.log(3), 0.0])
    assert np.allclose(ws.read_weight().cpu(), [0.75, 0.25], atol=1e-15)
    ws.set_log_weight([0.0, -np.inf])
    ws.add_log_weight([0.0, 5.0])
    assert ws.read_weight().tolist() == [1.0, 0.0]
    ws = WeightSet(4)
    ws.set_weight([2, 2, 2, 2])
    assert np.allclose(ws.read_weight().cpu(), 0.25, atol=1e-16)
    ws.set_equal_weight()
    ws.mul_weight([1, 1, 1, 3])
    assert np.allclose(ws.read_weight().cpu(), [1 / 6, 1 / 6, 1 / 6, 0.5], atol=1e-15)
    ws = WeightSet(3)
    ws.set_log_weight(np.log([0.5, 0.25, 0.25]))
    assert abs(ws.ess() - 8 / 3) < 1e-12
    ws = WeightSet(2)
    ws.set_log_weight([0.0, 0.0])
    assert np.allclose(ws.read_log_weight().cpu(), -math.log(2), atol=1e-15)
    with pytest.raises(_abi.SmcError):
        ws.set_log_weight([-np.inf, -np.inf])
    with pytest.raises(_abi.SmcError):
        ws.set_log_weight([0.0, np.nan])


@pytest.mark.parametrize("n", [1, 5, 255, 256, 257, 100000, 1 << 22])
def test_weights_vs_oracle(n):
    from paper_1306_5583_b200 import WeightSet
    rng = np.random.default_rng(n)
    v = rng.normal(0, 5, n)
    inc = rng.normal(0, 2, n)
    lw, w, ess = O.normalize_log(v)
    nc = O.nc_increment(lw, inc)
    ess2 = O.weights_update(O.W_ADD_LOG, lw, w, inc)
    ws = WeightSet(n)
    ws.set_log_weight(v)
    assert abs(ws.ess() - ess) <= 1e-12 * ess
    ws.add_log_weight(inc)
    st = ws.host_state()
    assert abs(st.ess - ess2) <= 1e-10 * ess2  # oracle: sequential sum over N; device: tree
    assert abs(st.nc_inc - nc) <= 1e-12 * max(1.0, abs(nc))
    np.testing.assert_allclose(ws.read_log_weight().cpu().numpy(), lw, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ws.read_weight().cpu().numpy(), w, rtol=1e-11, atol=1e-300)


def test_weighted_reduce_monitor():
    from paper_1306_5583_b200 import Sampler, StateMatrix, WeightSet, _abi
    n, m = 100003, 3
    rng = np.random.default_rng(4)
    vals = rng.normal(size=(n, m))
    v = rng.normal(0, 2, n)
    _, w, _ = O.normalize_log(v)
    ref = np.zeros(m)
    O.lib().orc_weighted_sum(w, vals, n, m, ref)
    ws = WeightSet(n)
    ws.set_log_weight(v)
    out = torch.zeros(m, dtype=torch.float64, device="cuda")
    buf = _abi.Workspace("cuda")
    b, nb = buf.get(_abi.lib().smc_weighted_reduce_workspace_bytes(n, m))
    g = torch.as_tensor(vals).cuda().contiguous()
    _abi.call("smc_weighted_reduce", _abi.ptr(g), m, m, _abi.ptr(ws.lw_raw), ws.state_ptr, n, _abi.ptr(out), b, nb,
              _abi.stream())
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-10, atol=1e-14)


def _obs(T=100, seed=1306):
    from paper_1306_5583_b200 import pf
    return pf.generate_observations(T, seed)


def test_pf_single_move_matches_oracle():
    from paper_1306_5583_b200 import pf
    n = 10000
    obs, _ = _obs(5)
    s = pf.make_sampler(n, "systematic", threshold=-1.0, seed=99)
    s.initialize(obs)
    st = O.Streams(n + 1, 99)
    x, llh = O.cv_init(n, st, obs[0])
    np.testing.assert_allclose(s.system.value.data.cpu().numpy(), x, rtol=1e-14, atol=1e-14)
    lw, w, ess = O.normalize_log(llh)
    assert abs(s.system.weight_set.ess() - ess) <= 1e-12 * ess
    s.iterate(1)
    incw = O.cv_move(x, st, obs[1])
    O.weights_update(O.W_ADD_LOG, lw, w, incw)
    np.testing.assert_allclose(s.system.value.data.cpu().numpy(), x, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(s.system.weight_set.read_log_weight().cpu().numpy(), lw, rtol=1e-11, atol=1e-11)
    assert s.system.rng_set.counters_host()[:n] == [int(c) for c in st.counters[:n]]


@pytest.mark.parametrize("scheme", ["systematic", "stratified", "multinomial", "residual", "residual_stratified",
                                    "residual_systematic"])
def test_pf_full_run_matches_oracle(scheme):
    """Config 1 (N=10^4, 100 obs, ESS<N/2): GPU RNG end to end vs the oracle."""
    from paper_1306_5583_b200 import pf
    n = 10000
    obs, _ = _obs(100)
    s = pf.make_sampler(n, scheme, threshold=0.5, seed=1306)
    s.initialize(obs)
    s.iterate(99)
    h = s.history()
    ref, xref, lwref = O.pf_run(n, 1306, scheme, 0.5, obs, want_state=True)
    assert np.array_equal(h["resampled"], ref[:, 1])
    # final state (the deferred resample copy is materialized on read) and log-weights
    np.testing.assert_allclose(s.system.value.data.cpu().numpy(), xref, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(s.system.weight_set.read_log_weight().cpu().numpy(), lwref, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(h["ess_over_n"], ref[:, 0], rtol=RTOL)
    np.testing.assert_allclose(h["pos.0"], ref[:, 2], rtol=RTOL, atol=1e-9)
    np.testing.assert_allclose(h["pos.1"], ref[:, 3], rtol=RTOL, atol=1e-9)
    assert abs(s.log_zconst - ref[-1, 4]) <= RTOL * abs(ref[-1, 4])


def test_pf_beats_observations_acceptance_6():
    from paper_1306_5583_b200 import pf
    wins = 0
    for seed in range(10):
        obs, truth = _obs(100, 100 + seed)
        s = pf.make_sampler(1000, "stratified", 0.5, seed=seed)
        s.initialize(obs)
        s.iterate(99)
        h = s.history()
        est = np.stack([h["pos.0"], h["pos.1"]], 1)
        wins += np.mean((est - truth[:, :2]) ** 2) < np.mean((obs - truth[:, :2]) ** 2)
    assert wins >= 9


def test_history_invariants_and_tsv(tmp_path):
    from paper_1306_5583_b200 import pf
    obs, _ = _obs(30)
    s = pf.make_sampler(4096, "stratified", 0.5, seed=3)
    s.initialize(obs)
    s.iterate(29)
    h = s.history()
    assert len(h["iter"]) == 30
    assert np.all((h["resampled"] == 1) == (h["ess_over_n"] < 0.5))
    text = s.write_tsv(tmp_path / "pf.est", ["seed=3"])
    lines = text.splitlines()
    assert lines[1].split("\t") == ["iter", "ess_over_n", "resampled", "accept.0", "pos.0", "pos.1"]
    assert len(lines) == 32
    s2 = pf.make_sampler(4096, "stratified", 0.5, seed=3)
    s2.initialize(obs)
    s2.iterate(29)
    assert s2.write_tsv(tmp_path / "b.est", ["seed=3"]) == text  # byte-identical reruns


def test_threshold_rules():
    from paper_1306_5583_b200 import pf
    obs, _ = _obs(10)
    for thr, expect in ((1.5, 1.0), (-1.0, 0.0)):
        s = pf.make_sampler(2000, "systematic", thr, seed=1)
        s.initialize(obs)
        s.iterate(9)
        assert np.all(s.history()["resampled"] == expect)


def test_statematrix_copy_simultaneous():
    from paper_1306_5583_b200 import StateMatrix
    m = StateMatrix(2, 3)
    m.data.copy_(torch.tensor([[1.0, 2, 3], [4, 5, 6]]))
    m.copy_particles([1, 0])
    assert m.data.tolist() == [[4, 5, 6], [1, 2, 3]]
    c = StateMatrix(3, 2, order="col")
    c.data.copy_(torch.tensor([[1.0, 2, 3], [4, 5, 6]]))
    c.copy_particles([0, 0, 2])
    assert c.read_state(0).tolist() == [1, 1, 3] and c.read_state(1).tolist() == [4, 4, 6]


@pytest.mark.parametrize("scheme,n", [("systematic", 10000), ("stratified", 4096), ("multinomial", 3000)])
def test_graph_replay_is_bit_identical_to_eager(scheme, n):
    """core.Sampler's CUDA-graph replay of iterate() runs the eager step's kernels in the
    same order: history, state, weights and log Z are bit-identical."""
    from paper_1306_5583_b200 import pf
    obs, _ = _obs(60)
    runs = []
    for graph in (False, "auto"):
        s = pf.make_sampler(n, scheme, threshold=0.5, seed=11)
        s.graph = graph
        s.graph_min_steps = 4
        s.initialize(obs)
        s.iterate(20)
        mid = s.history_array()  # a read between iterate() calls (flushes the fused monitor)
        s.iterate(17)
        s.iterate(21)
        runs.append((mid, s.history_array(), s.system.value.data.cpu().numpy(),
                     s.system.weight_set.read_log_weight().cpu().numpy(), s.log_zconst))
    assert getattr(s, "_gbuf", None) is not None and s._gbuf["graphs"], "graph mode did not engage"
    (m0, h0, x0, w0, z0), (m1, h1, x1, w1, z1) = runs
    assert np.array_equal(m0, m1) and np.array_equal(h0, h1)
    assert np.array_equal(x0, x1) and np.array_equal(w0, w1) and z0 == z1


def test_graph_replay_stops_at_the_last_observation():
    """iterate() past the data with graph='auto': the replayed pairs stop before the last
    observation and the eager remainder raises IndexError (no device-side fault)."""
    from paper_1306_5583_b200 import pf
    obs, _ = _obs(40)
    s = pf.make_sampler(4096, "systematic", threshold=0.5, seed=5)
    s.graph_min_steps = 4
    s.initialize(obs)
    with pytest.raises(IndexError):
        s.iterate(45)
    assert s.iteration == 39  # every observation was used, none past the end
    torch.cuda.synchronize()  # the context is still healthy
    assert s._gbuf["graphs"], "graph mode did not engage"
    h = s.history()
    assert np.all(np.isfinite(h["pos.0"]))


def test_graph_replay_follows_changed_scheme_and_threshold():
    """A cached graph must not replay an old scheme / threshold after the caller changes them."""
    from paper_1306_5583_b200 import pf
    from paper_1306_5583_b200.resample import _scheme
    obs, _ = _obs(60)
    runs = []
    for graph in (False, "auto"):
        s = pf.make_sampler(4096, "systematic", threshold=0.5, seed=13)
        s.graph = graph
        s.graph_min_steps = 4
        s.initialize(obs)
        s.iterate(20)
        s.system.resample_scheme = _scheme("multinomial")
        s.system.threshold = 0.9
        s.initialize(obs)
        s.iterate(30)
        runs.append((s.history_array(), s.log_zconst))
    assert np.array_equal(runs[0][0], runs[1][0]) and runs[0][1] == runs[1][1]


def test_invariants_shift_trapezoid_ais():
    """SPEC acceptance 8 invariant suites: log-weight shift invariance, trapezoid exactness on
    linear integrands, and AIS/SIS equivalence at threshold <= 0 (no resampling: the running
    log Z telescopes to log mean exp of each particle's accumulated increments)."""
    from paper_1306_5583_b200 import PathAccumulator, WeightSet, gmm
    rng = np.random.default_rng(9)
    v = rng.normal(0, 3, 5000)
    a, b = WeightSet(5000), WeightSet(5000)
    a.set_log_weight(v)
    b.set_log_weight(v + 123.456)
    np.testing.assert_allclose(a.read_weight().cpu().numpy(), b.read_weight().cpu().numpy(), rtol=1e-12, atol=0)
    assert abs(a.ess() - b.ess()) <= 1e-9 * a.ess()
    grid = np.linspace(0, 1, 11) ** 2
    pa = PathAccumulator(grid, 3.0 - 2.0 * grid)
    assert abs(pa.log_zconst - 2.0) < 1e-15  # integral of 3 - 2a over [0, 1]
    # no resampling and no MCMC: the particles stay prior draws and the increments sum to
    # (sum_t dalpha_t) llh_i = llh_i, so log Z telescopes to log mean_i exp(llh_i)
    y = gmm.generate_data(60, 21)
    s = gmm.make_sampler(4096, data=y, T=12, seed=8, threshold=0.0)
    s.mcmc_queue = []
    s.initialize()
    s.iterate(12)
    assert not np.any(s.history()["resampled"])
    llh = s.system.value.data[:, 13].cpu().numpy()
    m = llh.max()
    ais = m + np.log(np.mean(np.exp(llh - m)))
    assert abs(s.log_zconst - ais) <= 1e-10 * max(1.0, abs(ais)), (s.log_zconst, ais)


def test_pf_uniform_counter_move_is_bit_identical_to_counter_array():
    """smc_pf_move_uniform (every particle stream at one draw count, the count a kernel
    parameter) vs smc_pf_move on the counter array: same state, log-weights and counters,
    also across the 2^32 boundary of the counter's low word (the uniform path declines
    the step whose 16 draws would carry; smc_pf_move_uniform rejects such a count)."""
    from paper_1306_5583_b200 import _abi, pf
    n = 20000
    obs, _ = _obs(8)
    a = pf.make_sampler(n, "systematic", threshold=0.5, seed=7)
    b = pf.make_sampler(n, "systematic", threshold=0.5, seed=7)
    a.initialize(obs)
    b.initialize(obs)
    assert a.system.rng_set.uniform_count(n, 16) == 8
    start = (1 << 32) - 24  # moves at lo32 = 2^32-24, -16 (uniform), -8 (carry: array), 0, 8 (uniform)
    for s in (a, b):
        s.system.rng_set.counters.fill_(start)
    a.system.rng_set.advance_uniform(n, start, True)
    used = []
    for t in range(5):
        used.append(a.system.rng_set.uniform_count(n, 16) is not None)
        a.iterate(1)
        b.system.rng_set.counters  # drop the knowledge: b always runs the counter-array kernel
        b.iterate(1)
        assert torch.equal(a.system.value.data, b.system.value.data), t
        assert torch.equal(a.system.weight_set.read_log_weight(), b.system.weight_set.read_log_weight()), t
    assert used == [True, True, False, True, True]
    assert a.system.rng_set.counters_host()[:n] == b.system.rng_set.counters_host()[:n] == [start + 40] * n
    assert a.log_zconst == b.log_zconst
    # a count whose 16 draws carry is refused by the entry point itself
    v, w = a.system.value, a.system.weight_set
    ws, nb = pf._ws(a.system, n)
    with pytest.raises(_abi.SmcError):
        _abi.call("smc_pf_move_uniform", None, _abi.ptr(v.raw), None, None, _abi.ptr(w.lw_raw), n, 0, n, 7,
                  (1 << 32) - 15, v.obs_ptr(1), w.state_ptr, None, None, None, ws, nb, _abi.stream())


def test_lazy_uniform_counts_are_materialized_for_every_consumer():
    """After uniform-count moves the counter array lags the streams; a scalar draw, the
    counter readout and the next (counter-array) move all see the true counts."""
    from paper_1306_5583_b200 import pf
    from paper_1306_5583_b200.rng import RngStreamSet
    n = 1000
    obs, _ = _obs(8)
    s = pf.make_sampler(n, "systematic", threshold=0.5, seed=3)
    s.initialize(obs)
    s.iterate(3)
    rs = s.system.rng_set
    assert rs.uniform_count(n, 0) == 32  # init + 3 moves, 8 draws each
    x = rs.stream(5).uniform01()
    ref = RngStreamSet(n + 1, 3)
    ref.counters.fill_(32)
    assert x == ref.stream(5).uniform01()
    assert rs.uniform_count(n, 0) is None  # stream 5 left the common count
    c = rs.counters_host()
    assert c[5] == 33 and c[:5] == [32] * 5 and c[6:n] == [32] * (n - 6)
    s.iterate(1)  # the counter-array kernel from here on
    c = rs.counters_host()
    assert c[5] == 41 and c[:5] == [40] * 5 and c[6:n] == [40] * (n - 6)


@pytest.mark.parametrize("uniform", [True, False])
def test_warp_specialized_move_is_bit_identical(uniform):
    """k_pf_move_ws (Philox producer warps + Box-Muller consumer warps, draws handed over through a
    shared-memory ring) and the single-role k_pf_move compute the same arithmetic: identical state,
    log-weights, history and log Z, for the uniform-count and the counter-array move."""
    from paper_1306_5583_b200 import _abi, pf
    obs, _ = _obs(12)
    n = (1 << 20) + 77  # >= 4 blocks per SM (the path both kernels serve) and a partial last block
    runs = []
    for ws in (0, 1):
        _abi.call("smc_debug_set", 2, ws)  # SMC_DEBUG_MOVE_WS
        try:
            s = pf.make_sampler(n, "systematic", 0.5, seed=21)
            s.graph = False
            s.initialize(obs)
            if not uniform:
                _ = s.system.rng_set.counters  # materialized: the counter-array kernel from here on
            s.iterate(11)
            runs.append((s.history_array(), s.system.value.data.cpu().numpy(),
                         s.system.weight_set.read_log_weight().cpu().numpy(), s.log_zconst,
                         s.system.rng_set.counters_host()[:5]))
        finally:
            _abi.call("smc_debug_set", 2, 0)  # back to the default (single-role) move
    (h0, x0, w0, z0, c0), (h1, x1, w1, z1, c1) = runs
    assert np.array_equal(h0, h1) and np.array_equal(x0, x1) and np.array_equal(w0, w1) and z0 == z1 and c0 == c1
