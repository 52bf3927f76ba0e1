"""Run-time compiled user particle kernels (smc_user_compile / paper_1306_5583_b200.user):
the paper's particle filter written as plain user kernels must reproduce the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

PF_SRC = r'''
#include "smc_user.cuh"
__device__ double cv_llh(double xp, double yp, double xo, double yo)
{   // PAPER.md:1181-1191
    const double rx = 10 * (xp - xo), ry = 10 * (yp - yo);
    return -0.5 * (10 + 1) * (log(1 + rx * rx / 10) + log(1 + ry * ry / 10));
}
__device__ int cv_init_user(smc::Particle &p, unsigned long long iter, const double *obs)
{   // PAPER.md:1234-1255: draw order x, y, vx, vy
    p.state(0) = p.normal(0.0, 2.0);
    p.state(1) = p.normal(0.0, 2.0);
    p.state(2) = p.normal(0.0, 1.0);
    p.state(3) = p.normal(0.0, 1.0);
    p.slot(0) = cv_llh(p.state(0), p.state(1), obs[0], obs[1]);
    return 0;
}
SMC_USER_MOVE(cv_init_user)
'''

MOVE_SRC = r'''
#include "smc_user.cuh"
__device__ double cv_llh(double xp, double yp, double xo, double yo)
{
    const double rx = 10 * (xp - xo), ry = 10 * (yp - yo);
    return -0.5 * (10 + 1) * (log(1 + rx * rx / 10) + log(1 + ry * ry / 10));
}
__device__ int cv_move_user(smc::Particle &p, unsigned long long iter, const double *obs)
{   // PAPER.md:1297-1328, evaluation order x0 + ((0 + sd z) + delta x2)
    const double sp = sqrt(0.02), sv = sqrt(0.001);
    double x0 = p.state(0), x1 = p.state(1), x2 = p.state(2), x3 = p.state(3);
    x0 = x0 + (p.normal(0.0, sp) + 0.1 * x2);
    x1 = x1 + (p.normal(0.0, sp) + 0.1 * x3);
    x2 = x2 + p.normal(0.0, sv);
    x3 = x3 + p.normal(0.0, sv);
    p.state(0) = x0; p.state(1) = x1; p.state(2) = x2; p.state(3) = x3;
    p.slot(0) = cv_llh(x0, x1, obs[0], obs[1]);
    return 0;
}
SMC_USER_MOVE(cv_move_user)
'''

MON_SRC = r'''
#include "smc_user.cuh"
__device__ void pos(const smc::Particle &p, unsigned long long iter, const double *prm, double *out)
{
    out[0] = p.state(0);
    out[1] = p.state(1);
}
SMC_USER_EVAL(pos)
'''


def _user_pf(n, scheme, seed, obs):
    from paper_1306_5583_b200 import Sampler, StateMatrix, user
    o = torch.as_tensor(obs, dtype=torch.float64).cuda().contiguous()
    s = Sampler(n, scheme, 0.5, seed, value=StateMatrix(n, 4))
    s.set_init(user.compile_move(PF_SRC, 1, params=o, post=user.set_scratch_log_weight(0)))
    s.add_move(user.compile_move(MOVE_SRC, 1, params=lambda it, sysm: o[it], post=user.add_scratch_log_weight(0)))
    s.set_monitor("pos", 2, user.compile_monitor(MON_SRC, 2))
    return s


@pytest.mark.parametrize("scheme", ["systematic", "residual"])
def test_user_kernel_pf_matches_oracle(scheme):
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(40, 7)
    n = 4096
    s = _user_pf(n, scheme, 1306, obs)
    s.initialize()
    s.iterate(39)
    h = s.history()
    ref, xref, _ = O.pf_run(n, 1306, scheme, 0.5, obs, want_state=True)
    assert np.array_equal(h["resampled"], ref[:, 1])
    np.testing.assert_allclose(h["ess_over_n"], ref[:, 0], rtol=1e-6)
    np.testing.assert_allclose(h["pos.0"], ref[:, 2], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(h["pos.1"], ref[:, 3], rtol=1e-6, atol=1e-9)
    assert abs(s.log_zconst - ref[-1, 4]) <= 1e-6 * abs(ref[-1, 4])
    np.testing.assert_allclose(s.system.value.data.cpu().numpy(), xref, rtol=1e-8, atol=1e-9)


def test_user_kernel_matches_builtin_pf():
    """Same seed, same draws: the generic path and the fused built-in kernels agree."""
    from paper_1306_5583_b200 import pf
    obs, _ = pf.generate_observations(20, 3)
    a = _user_pf(2048, "stratified", 9, obs)
    a.initialize()
    a.iterate(19)
    b = pf.make_sampler(2048, "stratified", 0.5, 9)
    b.initialize(obs)
    b.iterate(19)
    ha, hb = a.history(), b.history()
    assert np.array_equal(ha["resampled"], hb["resampled"])
    np.testing.assert_allclose(ha["pos.0"], hb["pos.0"], rtol=1e-9, atol=1e-12)
    assert abs(a.log_zconst - b.log_zconst) < 1e-9 * abs(b.log_zconst)


def test_user_rng_bit_exact_and_col_major():
    """Draws through smc::Particle equal the library's stream draws bit for bit;
    column-major state addressing; exact acceptance counts."""
    from paper_1306_5583_b200 import ParticleSystem, StateMatrix, user
    src = r'''
    #include "smc_user.cuh"
    __device__ int k(smc::Particle &p, unsigned long long iter, const double *prm)
    {
        p.state(0) = p.u01();
        p.state(1) = p.normal(prm[0], prm[1]);
        p.state(2) = p.gamma(prm[2], 1.0);
        return (p.id % 3) == 0;
    }
    SMC_USER_MOVE(k)
    '''
    n = 5000
    v = StateMatrix(n, 3, order="col")
    sysm = ParticleSystem(v, n, seed=77)
    op = user.compile_move(src, params=torch.tensor([0.0, 1.0, 0.7], dtype=torch.float64, device="cuda"))
    acc = op(0, sysm)
    assert int(acc.item()) == (n + 2) // 3
    st = O.Streams(n + 1, 77)
    x = v.data.cpu().numpy()
    for i in (0, 1, 2, 1234, n - 1):
        u, z, g = st.u01(i), st.normal(i), st.gamma(i, 0.7)  # the kernel's draw order
        assert x[0, i] == u  # u01: bit-exact
        assert abs(x[1, i] - z) <= 1e-14 * max(1.0, abs(z))  # log differs from glibc by <= 1 ulp
        assert abs(x[2, i] - g) <= 1e-12 * g
    assert sysm.rng_set.counters_host()[1234] == int(st.counters[1234])


def test_compile_errors_are_reported():
    from paper_1306_5583_b200 import _abi, user
    with pytest.raises(_abi.SmcError, match="error"):
        user.UserKernel('#include "smc_user.cuh"\n__device__ int f(smc::Particle &p) { return undefined_x; }\n'
                        'SMC_USER_MOVE(f)\n')
    with pytest.raises(_abi.SmcError, match="SMC_USER_MOVE"):
        user.UserKernel('#include "smc_user.cuh"\n__device__ int f() { return 0; }\n')
    with pytest.raises(ValueError):
        user.compile_monitor(MOVE_SRC, 2)
