"""SPEC's TRIVIAL / rejection cases of the sampler and the resampler on the device
(empty inputs)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_sampler_rejects_zero_particles():
    from paper_1306_5583_b200 import pf
    with pytest.raises(ValueError):
        pf.make_sampler(0, "systematic", 0.5, seed=1)  # N = 0 -> rejection


def test_fresh_sampler_equal_weights_and_iterate_zero_is_noop():
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(5, 3)
    s = pf.make_sampler(100, "systematic", 0.5, seed=3)
    ws = s.system.weight_set
    assert abs(ws.ess() / 100 - 1.0) < 1e-12  # sampler_new(100): ESS/N = 1 before any iteration
    s.initialize(obs)
    h0 = {k: np.array(v) for k, v in s.history().items()}
    x0 = s.system.value.data.clone()
    s.iterate(0)  # n = 0 -> no-op
    h1 = s.history()
    assert s.iteration == 0 and all(np.array_equal(h0[k], np.array(h1[k])) for k in h0)
    assert torch.equal(x0, s.system.value.data)


def test_initialize_without_init_and_empty_monitor_rejected():
    from paper_1306_5583_b200 import core, pf
    s = core.Sampler(10, "systematic", 0.5, 1, value=pf.CVState(10, "cuda"))
    with pytest.raises(RuntimeError):
        s.initialize()  # missing init op -> rejection
    with pytest.raises(ValueError):
        s.set_monitor("empty", 0, pf.cv_monitor(2))  # m = 0 -> rejection


def test_resample_empty_input_rejected():
    from paper_1306_5583_b200 import _abi, resample
    with pytest.raises((_abi.SmcError, ValueError)):
        resample("systematic", torch.empty(0, dtype=torch.float64, device="cuda"),
                 u=torch.tensor([0.5], dtype=torch.float64, device="cuda"))


def test_after_resampling_weights_equal():
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(4, 5)
    s = pf.make_sampler(4096, "systematic", 1.5, seed=5)  # resample every iteration
    s.initialize(obs)
    s.iterate(2)
    w = s.system.weight_set.read_weight().cpu().numpy()
    assert np.all(w == w[0]) and abs(w.sum() - 1.0) < 1e-12  # after resampling ESS/N = 1


def test_first_failing_particle_index_is_reported():
    """a failing per-particle kernel reports the FIRST failing particle's
    index (the lowest, whatever order the threads ran in) next to the error code."""
    from paper_1306_5583_b200 import WeightSet, _abi
    n = 100000
    v = torch.zeros(n, dtype=torch.float64, device="cuda")
    v[[77777, 4242, 99999]] = float("nan")
    ws = WeightSet(n)
    ws.set_log_weight(v, check=False)
    with pytest.raises(_abi.SmcError) as e:
        ws.raise_if_failed()
    assert e.value.code == -3 and e.value.index == 4242 and "first failing particle 4242" in str(e.value)
    ws.set_log_weight(torch.zeros(n, dtype=torch.float64, device="cuda"))  # cleared: healthy again


def test_resample_reports_first_bad_weight_and_negative_count():
    from paper_1306_5583_b200 import _abi, replication_to_parents, resample
    n = 50000
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    w[31337] = -1.0 / n
    w[40000] = float("nan")
    with pytest.raises(_abi.SmcError) as e:
        resample("stratified", w, u=torch.rand(n, dtype=torch.float64, device="cuda"))
    assert e.value.code == -2 and e.value.index == 31337
    c = torch.ones(n, dtype=torch.int32, device="cuda")
    c[[12345, 23456]] = -1
    c[[1, 2]] = 2
    with pytest.raises(_abi.SmcError) as e:
        replication_to_parents(c)
    assert e.value.code == -5 and e.value.index == 12345


def test_pf_move_reports_the_particle_whose_weight_failed():
    """A non-finite observation makes every particle's likelihood NaN: particle 0 is the first."""
    from paper_1306_5583_b200 import _abi, pf
    obs, _ = pf.generate_observations(4, 3)
    obs[2, 0] = float("nan")
    s = pf.make_sampler(5000, "systematic", 0.5, seed=3)
    s.initialize(obs)
    with pytest.raises(_abi.SmcError) as e:
        s.iterate(2)
    assert e.value.code == -3 and e.value.index == 0
