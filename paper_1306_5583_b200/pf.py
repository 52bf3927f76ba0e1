"""The paper's particle filter on the device (mirror of smckit example-pf).

Almost-constant-velocity tracking: X = (x_pos, y_pos,
x_vel, y_vel) as an N x 4 row-major StateMatrix, Student-t
(nu = 10) observation likelihood scaled by 10.

    sampler = make_sampler(N, scheme="systematic", threshold=0.5, seed=1306)
    sampler.initialize(obs)          # obs: (T, 2) array or a pf.data path
    sampler.iterate(obs.shape[0] - 1)
    sampler.history()["pos.0"]       # filtered x_pos means

``cv_init``/``cv_move`` are fused device kernels: the move updates the state,
draws its four normals from the particle's own stream, evaluates the
likelihood and applies add_log_weight with the one-pass lse/ESS partials.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _abi
from .core import ROW_MAJOR, Sampler, StateMatrix
from .exec import MonitorEval, ParticleKernelOp
from .resample import ResampleScheme
from .rng import RngStreamSet

__all__ = ["CVState", "cv_init", "cv_move", "cv_monitor", "make_sampler", "cv_log_likelihood",
           "generate_observations", "load_observations", "write_observations", "DATA_NUM"]

DATA_NUM = 100


class CVState(StateMatrix):
    """StateMatrix<RowMajor, 4, double> + the observations."""

    # cv_move gathers x_in[parents[i]] into the second buffer, so a resample only
    # builds the parent map and never copies rows itself (see smc_pf_move).
    defer_copy = True

    def __init__(self, size, device="cuda"):
        super().__init__(size, 4, ROW_MAJOR, device)
        self.obs = None  # (T, 2) float64 on the device
        self.graph_obs = None  # CUDA-graph replay: the step's observation, gathered by a device index

    def read_data(self, source):
        if isinstance(source, (str, os.PathLike)):
            arr = load_observations(source)
        else:
            arr = np.asarray(source, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] != 2:
            raise ValueError("observations must be (T, 2)")
        self.obs = torch.as_tensor(arr, dtype=torch.float64).to(self.device).contiguous()

    def obs_ptr(self, t):
        if self.graph_obs is not None:
            return ctypes.c_void_p(self.graph_obs.data_ptr())
        if self.obs is None:
            raise RuntimeError("no observations loaded")
        if not 0 <= t < self.obs.shape[0]:
            raise IndexError(f"no observation for iteration {t}")
        return ctypes.c_void_p(self.obs.data_ptr() + 16 * t)


def _ws(system, n):
    ws = getattr(system, "_pf_ws", None)
    if ws is None:
        ws = system._pf_ws = _abi.Workspace(system.device)
    return ws.get(_abi.lib().smc_pf_workspace_bytes(n))


def cv_init(system, param=None):
    """cv_init: read data if given, draw the prior, set_log_weight(llh_0)."""
    v = system.value
    if param is not None:
        v.read_data(param)
    n = system.size
    ws, nb = _ws(system, n)
    w = system.weight_set
    v.pending = None  # the prior draw overwrites every row
    shard = system.shard
    rs = system.rng_set
    u = rs.uniform_count(n, 0)
    _abi.call("smc_pf_init", _abi.ptr(v.raw), _abi.ptr(w.lw_raw), n, system.stream_base, rs.seed,
              _abi.ptr(rs.counters), v.obs_ptr(0), w.state_ptr,
              None if shard is None else _abi.ptr(shard.partial), ws, nb, _abi.stream())
    if u is not None:  # every particle stream drew 8: still uniform (and written)
        rs.advance_uniform(n, (u + 8) % (1 << 64), True)
    if shard is not None:  # global normalization: allgather the shard partials, combine in rank order
        shard.combine(w, 0, True)  # SMC_W_SET_LOG
    return None  # acceptance "bares no meaning"


def _cv_move_kernel(iter_, system):
    v = system.value
    n = system.size
    ws, nb = _ws(system, n)
    w = system.weight_set
    # a pending fused "pos" monitor of the previous iteration is reduced by this launch
    mon = system.take_pending_monitor("pos")
    shard = system.shard
    rs = system.rng_set
    # every particle stream at one draw count (the PF's own streams advance in lockstep):
    # the kernel takes the count as a scalar and leaves the counter array alone
    u0 = rs.uniform_count(n, 0)
    u = rs.uniform_count(n, 16)  # the kernel's precomputed table covers 16 draws without a carry
    if system.stream_base + n > 1 << 32:  # ... and stream indices below 2^32
        u = None
    fn, ctr = ("smc_pf_move", _abi.ptr(rs.counters)) if u is None else ("smc_pf_move_uniform", u)
    common = (_abi.ptr(w.lw_raw), n, system.stream_base, system.n_total, rs.seed, ctr, v.obs_ptr(iter_),
              w.state_ptr, None, mon, None if shard is None else _abi.ptr(shard.partial), ws, nb, _abi.stream())
    if v.pending is not None:  # fold the last resample's copy into this move (double buffer)
        parents, gate = v.pending
        v.pending = None
        _abi.call(fn, _abi.ptr(v.raw), _abi.ptr(v.alt()), _abi.ptr(parents), gate, *common)
        v.swap()
    else:
        _abi.call(fn, None, _abi.ptr(v.raw), None, None, *common)
    if u0 is not None:  # every particle stream drew 8 (the array written iff it was passed)
        rs.advance_uniform(n, (u0 + 8) % (1 << 64), u is None)
    if shard is not None:  # global add_log_weight + the fused monitor of the previous iteration
        shard.combine(w, 1, True, mon)  # SMC_W_ADD_LOG
    return None


def cv_move():
    """cv_move as a ParticleKernelOp; post add_log_weight is fused.
    graph_safe: every launch is stream-ordered device work with fixed addresses, so the
    sampler may capture and replay it in a CUDA graph (core.Sampler._iterate_graph)."""
    op = ParticleKernelOp(_cv_move_kernel, name="cv_move")
    op.graph_safe = True
    return op


def cv_monitor(dim=2):
    """Monitor of (x_pos, y_pos) (dim=4 returns all columns).

    With dim=2 it is fusable: the next cv_move reduces it from the state it
    loads anyway (``fused_with="cv_move"``); the sampler falls back to the
    standalone weighted reduction whenever the history is read first."""
    ev = MonitorEval(lambda it, system: system.value.column_view(0, dim), dim)
    if dim == 2:
        ev.fused_with = "cv_move"
    return ev


def make_sampler(n, scheme=ResampleScheme.Systematic, threshold=0.5, seed=0, device="cuda", monitor_dim=2,
                 shard=None):
    """The paper's main(): sampler, init, move, 'pos' monitor.
    shard: a dist.Shard to run this as one rank of a multi-GPU filter (n particles per rank)."""
    s = Sampler(n, scheme, threshold, seed, value=CVState(n, device), device=device, shard=shard)
    s.set_init(cv_init)
    s.add_move(cv_move(), False)
    s.set_monitor("pos", monitor_dim, cv_monitor(monitor_dim))
    return s


def cv_log_likelihood(xpos, ypos, xobs, yobs):
    """Host restatement for documentation / tiny checks."""
    import math

    scale, nu = 10.0, 10.0
    lx = scale * (xpos - xobs)
    ly = scale * (ypos - yobs)
    lx = math.log(1 + lx * lx / nu)
    ly = math.log(1 + ly * ly / nu)
    return -0.5 * (nu + 1) * (lx + ly)


def generate_observations(n=DATA_NUM, seed=1306, device="cuda"):
    """Simulate the model from stream 0 of
    RngStreamSet(1, seed): X_0 ~ N(0, diag(4,4,1,1)); X_t = A X_{t-1} + V;
    Y_t = pos + 0.1 * t_10, with t = Z / sqrt(G / nu), G = 2 Gamma(nu / 2).
    Returns (obs (n,2), truth (n,4)) as numpy arrays.  Draws run on the device."""
    st = RngStreamSet(1, seed, device).stream(0)
    nu = 10.0
    x = np.empty(4)
    truth = np.empty((n, 4))
    obs = np.empty((n, 2))
    sd_pos, sd_vel, delta = 0.02 ** 0.5, 0.001 ** 0.5, 0.1
    for t in range(n):
        if t == 0:
            x[0] = st.normal(0.0, 2.0)
            x[1] = st.normal(0.0, 2.0)
            x[2] = st.normal(0.0, 1.0)
            x[3] = st.normal(0.0, 1.0)
        else:
            x[0] = x[0] + (st.normal(0.0, sd_pos) + delta * x[2])
            x[1] = x[1] + (st.normal(0.0, sd_pos) + delta * x[3])
            x[2] = x[2] + st.normal(0.0, sd_vel)
            x[3] = x[3] + st.normal(0.0, sd_vel)
        truth[t] = x
        for k in range(2):
            z = st.normal(0.0, 1.0)
            g = 2.0 * st.gamma(nu / 2.0, 1.0)
            obs[t, k] = x[k] + 0.1 * (z / (g / nu) ** 0.5)
    return obs, truth


def write_observations(path, obs, truth=None):
    """pf.data: T lines 'x y' (%.17g); optional .truth sibling."""
    with open(path, "w") as f:
        for a, b in obs:
            f.write(f"{a:.17g} {b:.17g}\n")
    if truth is not None:
        with open(str(path) + ".truth", "w") as f:
            for row in truth:
                f.write(" ".join(f"{v:.17g}" for v in row) + "\n")


def load_observations(path):
    """Whitespace-separated floats, two per line; errors name the line."""
    rows = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            if len(parts) != 2:
                raise ValueError(f"{path}:{ln}: expected 2 values, got {len(parts)}")
            try:
                rows.append([float(parts[0]), float(parts[1])])
            except ValueError as e:
                raise ValueError(f"{path}:{ln}: {e}") from None
    return np.asarray(rows, dtype=np.float64)
