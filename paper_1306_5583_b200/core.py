"""Sampler / ParticleSystem / StateMatrix on the device (mirror of smckit.core).

One ``Sampler.iterate()`` issues, with no host synchronization:

  move queue (device kernels; the PF move fuses add_log_weight + lse/ESS)
  -> smc_ess_decide         (device flag; history ess_over_n / resampled)
  -> smc_resample           (gated by the flag: counts, parent map and the
                             in-place row copy of the state matrix)
  -> set_equal_weight       (gated)
  -> mcmc queue
  -> monitors / path        (fused weighted reductions into the device history)

The history lives in a device tensor and is read back lazily (``history()``,
``write_tsv()``), so a run of many iterations costs one sync at the end.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _abi
from .exec import MonitorEval, PathEval, ParticleKernelOp, apply_monitor_eval, apply_path_eval, apply_move
from .resample import ResampleScheme, Resampler, _scheme
from .rng import RngStreamSet
from .weights import WeightSet

__all__ = ["StateMatrix", "ParticleSystem", "SingleParticleView", "Sampler", "MonitorRecord",
           "PathAccumulator", "NormalizingConstant", "ROW_MAJOR", "COL_MAJOR", "nc_add_log_weight", "sampler_new"]

ROW_MAJOR, COL_MAJOR = "row", "col"


class StateMatrix:
    """N x D float64 state (PAPER.md:714-726 RowMajor/ColMajor tag).

    Row-major storage puts one particle in one contiguous row, which the
    resampling kernel copies in place with a single 256-bit load/store when
    D == 4 (the PF).  Column-major is D contiguous columns.
    """

    def __init__(self, size, dim, order=ROW_MAJOR, device="cuda"):
        if order not in (ROW_MAJOR, COL_MAJOR):
            raise ValueError("order must be 'row' or 'col'")
        _abi.require_cuda()
        self.size, self.dim, self.order = int(size), int(dim), order
        self.device = torch.device(device)
        shape = (self.size, self.dim) if order == ROW_MAJOR else (self.dim, self.size)
        self._bufs = [torch.zeros(shape, dtype=torch.float64, device=self.device), None]
        self._cur = 0
        # A resample's copy may be deferred: (parents, gate) that the next gathering
        # kernel (or materialize()) applies "as simultaneous".
        self.pending = None

    # -- storage --------------------------------------------------------------
    @property
    def data(self):
        """The state (any deferred resample copy applied first)."""
        self.materialize()
        return self._bufs[self._cur]

    @data.setter
    def data(self, t):
        self.pending = None
        self._bufs[self._cur] = t

    @property
    def raw(self):
        """Current buffer WITHOUT applying a pending copy (for gathering kernels)."""
        return self._bufs[self._cur]

    def alt(self):
        """The second buffer of the double-buffered state (allocated on first use)."""
        o = 1 - self._cur
        if self._bufs[o] is None or self._bufs[o].shape != self._bufs[self._cur].shape:
            self._bufs[o] = torch.empty_like(self._bufs[self._cur])
        return self._bufs[o]

    def swap(self):
        self._cur = 1 - self._cur

    def materialize(self):
        """Apply a deferred resample copy in place (sources and destinations are disjoint)."""
        if self.pending is None:
            return
        parents, gate = self.pending
        self.pending = None
        self.copy_inplace(parents, gate)

    # element / column access
    def _check(self, i, pos):
        if not (0 <= i < self.size and 0 <= pos < self.dim):
            raise IndexError("state index out of range")

    def state(self, i, pos):
        self._check(i, pos)
        return float(self.data[i, pos] if self.order == ROW_MAJOR else self.data[pos, i])

    def set_state(self, i, pos, v):
        self._check(i, pos)
        if self.order == ROW_MAJOR:
            self.data[i, pos] = v
        else:
            self.data[pos, i] = v

    def read_state(self, pos):
        if not 0 <= pos < self.dim:
            raise IndexError("column out of range")
        return (self.data[:, pos] if self.order == ROW_MAJOR else self.data[pos]).clone()

    def read_state_matrix(self, order=ROW_MAJOR):
        m = self.data if self.order == ROW_MAJOR else self.data.t()
        return m.contiguous().clone() if order == ROW_MAJOR else m.t().contiguous().clone()

    def column_view(self, first, count):
        """(vals, ld) for monitors: columns first..first+count-1 without a copy."""
        if self.order == ROW_MAJOR:
            return self.data.view(-1)[first:], self.dim
        if count != 1:
            raise ValueError("column-major monitors take one column per evaluator")
        return self.data[first], 1

    # copies
    def copy_particles(self, parents):
        """Rows j <- rows parents[j], simultaneously (out of place: safe for any map)."""
        p = torch.as_tensor(parents, dtype=torch.int32).to(self.device).contiguous()
        if p.numel() != self.size:
            raise ValueError("parents length != size")
        if self.size and (int(p.min()) < 0 or int(p.max()) >= self.size):
            raise IndexError("parent index out of range")
        if self.order == ROW_MAJOR:
            out = torch.empty_like(self.data)
            _abi.call("smc_gather_rows", _abi.ptr(out), _abi.ptr(self.data), 8 * self.dim, _abi.ptr(p),
                      self.size, _abi.stream())
        else:
            out = torch.empty_like(self.data)
            for c in range(self.dim):
                _abi.call("smc_gather_rows", _abi.ptr(out[c]), _abi.ptr(self.data[c]), 8, _abi.ptr(p), self.size,
                          _abi.stream())
        self.data = out

    def resample_rows(self):
        """(rows_ptr, row_bytes) for the fused in-place copy in smc_resample, or None."""
        if self.order == ROW_MAJOR:
            return ctypes.c_void_p(self.data.data_ptr()), 8 * self.dim
        return None

    # A value collection whose next move kernel gathers x_in[parents[i]] (double
    # buffering) sets this: the sampler then only produces the parent map.
    defer_copy = False

    def copy_inplace(self, parents, gate=None):
        """In-place copy for a ParentVector (sources and destinations are disjoint)."""
        buf = self.raw
        if self.order == ROW_MAJOR:
            _abi.call("smc_copy_rows_inplace", ctypes.c_void_p(buf.data_ptr()), 8 * self.dim,
                      _abi.ptr(parents), self.size, gate, _abi.stream())
        else:
            for c in range(self.dim):
                _abi.call("smc_copy_rows_inplace", ctypes.c_void_p(buf[c].data_ptr()), 8, _abi.ptr(parents),
                          self.size, gate, _abi.stream())


class ParticleSystem:
    """value + WeightSet + RngStreamSet(N + 1) + resampling policy."""

    def __init__(self, value, size, scheme=ResampleScheme.Stratified, threshold=0.5, seed=0, device="cuda",
                 shard=None):
        self.value = value
        self.size = int(size)
        # shard: dist.Shard when this system is one rank's slice of a multi-GPU system
        self.shard = shard
        self.n_total = shard.n_total if shard is not None else self.size
        self.stream_base = shard.base if shard is not None else 0
        self.device = torch.device(device)
        self.weight_set = WeightSet(self.size, self.device, check=False)
        self.rng_set = RngStreamSet(self.size + 1, seed, self.device)
        self.resample_scheme = _scheme(scheme)
        self.threshold = float(threshold)
        self.parents = torch.arange(self.size, dtype=torch.int32, device=self.device)
        self.resampler = Resampler(self.size, self.device)
        self.pending_monitors = {}  # name -> device address a fused move kernel writes into

    def rng(self, i):
        return self.rng_set.stream(i)

    def take_pending_monitor(self, name):
        """Device address for a monitor the calling move kernel reduces in passing (or None)."""
        p = self.pending_monitors.pop(name, None)
        return None if p is None else ctypes.c_void_p(p[0])


class SingleParticleView:
    """Handle on particle ``id``.  Host-side convenience only:
    device kernels address their particle by thread index instead."""

    def __init__(self, id_, system):
        self.id = int(id_)
        self.system = system

    def state(self, pos):
        return self.system.value.state(self.id, pos)

    def set_state(self, pos, v):
        self.system.value.set_state(self.id, pos, v)

    def rng(self):
        return self.system.rng(self.id)


class MonitorRecord:
    """name, dim m, and the per-iteration estimates."""

    def __init__(self, name, dim, eval_):
        self.name, self.dim, self.eval = name, int(dim), eval_


class PathAccumulator:
    """grids alpha_t, integrands U_t, trapezoid log Z."""

    def __init__(self, grids=(), integrands=()):
        self.grids = list(grids)
        self.integrands = list(integrands)

    @property
    def log_zconst(self):
        g, u = self.grids, self.integrands
        return float(sum(0.5 * (g[t] - g[t - 1]) * (u[t] + u[t - 1]) for t in range(1, len(g))))


class NormalizingConstant:
    """Running log Z = sum_t log sum_i W_{t-1,i} exp(incw_{t,i}).

    Lives in the device weight record (smc_wstate.log_zconst); this is a view."""

    def __init__(self, weight_set):
        self.weight_set = weight_set

    @property
    def log_zconst(self):
        return self.weight_set.log_zconst


def nc_add_log_weight(nc, incw, weight_set):
    """log_zconst += log sum_i W_i exp(incw_i) over the current (pre-update)
    weights; the weights themselves are not changed.  (The samplers fuse this into their
    add_log_weight pass -- ``WeightSet.add_log_weight(incw, accumulate_nc=True)``; this
    standalone form runs the same kernels on a scratch copy and keeps only the increment.)"""
    ws = weight_set if weight_set is not None else nc.weight_set
    v = torch.as_tensor(incw, dtype=torch.float64, device=ws.device).contiguous()
    if v.numel() != ws.size:
        raise ValueError(f"expected {ws.size} increments, got {v.numel()}")
    lw, st = ws.lw_raw.clone(), ws.state.clone()
    buf, nb = ws._ws.get(_abi.lib().smc_weights_workspace_bytes(ws.size))
    _abi.call("smc_weights_update", 1, _abi.ptr(lw), _abi.ptr(v), ws.size, ctypes.c_void_p(st.data_ptr()), 1, buf,
              nb, _abi.stream())  # SMC_W_ADD_LOG with the NC increment
    off = _abi.WSTATE_OFF["log_zconst"]
    ws.state[off:off + 8].copy_(st[off:off + 8])


def sampler_new(N, scheme=None, threshold=0.5, **kw):
    """``sampler_new(N, scheme = Stratified, threshold = 0.5)``."""
    return Sampler(N, ResampleScheme.Stratified if scheme is None else scheme, threshold, **kw)


class Sampler:
    """SMC sampler.

    ``Sampler(N, scheme=Stratified, threshold=0.5, seed=0, value=...)``; the
    value collection defaults to an N x 1 StateMatrix.
    """

    def __init__(self, size, scheme=ResampleScheme.Stratified, threshold=0.5, seed=0, value=None, device="cuda",
                 shard=None):
        size = int(size)
        if size < 1:
            raise ValueError("sampler needs N >= 1")
        _abi.require_cuda()
        self.device = torch.device(device)
        if value is None:
            value = StateMatrix(size, 1, device=self.device)
        if shard is not None and not getattr(value, "defer_copy", False):
            raise ValueError("a sharded sampler needs a value collection whose move gathers (defer_copy)")
        self.system = ParticleSystem(value, size, scheme, threshold, seed, self.device, shard)
        self.init_op = None
        self.move_queue = []
        self.mcmc_queue = []
        self.monitors = {}
        self.path = None
        self._hist = None
        self._rows = 0
        self._cols = None
        self._path_grid = []
        self.iteration = -1
        self._ws = _abi.Workspace(self.device)
        self._mon_out = None

    # -- configuration -------------------------------------
    @property
    def size(self):
        return self.system.size

    @property
    def particle(self):
        return self.system

    def set_init(self, op):
        self.init_op = op
        return self

    init = set_init

    def add_move(self, op, append=False):
        if not append:
            self.move_queue = []
        self.move_queue.append(op)
        return self

    move = add_move

    def add_mcmc(self, op, append=False):
        if not append:
            self.mcmc_queue = []
        self.mcmc_queue.append(op)
        return self

    mcmc = add_mcmc

    def set_monitor(self, name, dim, eval_):
        if int(dim) < 1:
            raise ValueError("a monitor needs dimension m >= 1")  # SPEC.md:409 (empty monitor disallowed)
        if not isinstance(eval_, MonitorEval):
            eval_ = MonitorEval(eval_, dim)
        self.monitors[name] = MonitorRecord(name, dim, eval_)
        return self

    monitor = set_monitor

    def set_path(self, eval_):
        self.path = eval_ if isinstance(eval_, PathEval) else PathEval(eval_)
        return self

    path_sampling = set_path

    # -- history layout -----------------------------------------
    def _layout(self):
        cols = ["ess_over_n", "resampled"]
        nacc = max(len(self.move_queue) + len(self.mcmc_queue), 0)
        cols += [f"accept.{k}" for k in range(nacc)]
        if self.path is not None:
            cols += ["path.grid", "path.integrand"]
        for name, rec in self.monitors.items():
            cols += [f"{name}.{j}" for j in range(rec.dim)]
        self._cols = cols
        self._col = {c: k for k, c in enumerate(cols)}

    def _row(self, t):
        if self._hist is None or t >= self._hist.shape[0]:
            if self._hist is not None:
                self.flush()  # pending monitor addresses point into the old buffer
            cap = max(128, 2 * (t + 1))
            h = torch.zeros((cap, len(self._cols)), dtype=torch.float64, device=self.device)
            if self._hist is not None:
                h[: self._hist.shape[0]] = self._hist
            self._hist = h
        self._rows = max(self._rows, t + 1)
        return self._hist[t]

    # -- the loop -------------------------------------------
    def initialize(self, param=None, check=True):
        if self.init_op is None:
            raise RuntimeError("initialize: no init operation set")
        self._layout()
        self.system.pending_monitors.clear()
        if hasattr(self.system.value, "pending"):
            self.system.value.pending = None
        if self._hist is not None and self._hist.shape[1] == len(self._cols):
            self._hist.zero_()  # keep the buffer (and so any captured CUDA graph) across runs
        else:
            self._hist = None
        self._rows = 0
        self._path_grid = []
        sysm = self.system
        sysm.weight_set.set_equal_weight_if(None, sysm.n_total)
        row = self._row(0)
        acc = self.init_op(sysm, param) if not isinstance(self.init_op, ParticleKernelOp) \
            else apply_move(self.init_op, sysm, 0)
        del acc
        self.iteration = 0
        self._after_moves(0, row, [])
        if check:
            self.check()

    def iterate(self, n=1, check=True):
        if self.iteration < 0:
            raise RuntimeError("iterate: sampler not initialized")
        n = int(n)
        if n >= self.graph_min_steps and self._graph_ok():
            n = self._iterate_graph(n)  # whole pairs of steps replayed; returns the steps left
        for _ in range(n):
            self._step()
        if check and n >= 0:
            self.check()

    def _step(self):
        t = self.iteration + 1
        row = self._row(t)
        self._mark("move", 0)
        accs = [apply_move(op, self.system, t) for op in self.move_queue]
        self._mark("move", 1)
        self.iteration = t
        self._after_moves(t, row, accs)

    # -- CUDA-graph replay of iterate() -----------------------------------------
    # A step whose every launch is graph-safe (the built-in PF: cv_move with its fused
    # "pos" monitor, the ESS rule, the device-gated resample, set_equal_weight_if) is
    # captured ONCE as a CUDA graph of two steps and replayed: no Python and no per-launch
    # host work in the loop (launch-bound at small N).  What varies per step
    # lives on the device: the iteration index `t` (a counter the graph increments), the
    # observation (gathered by t into a fixed buffer), and the history row, written into one
    # of two fixed staging rows and copied into the history by t once the next move has
    # added the fused monitor.  Two steps per graph because the state is double-buffered.
    # The kernels and their order are exactly the eager step's: results are bit-identical.
    # The first capture in a process costs ~80 ms of one-time driver / allocator setup (later
    # captures ~1 ms); replay saves ~20 % per step at N = 10^4 (the GPU-side chain of ~14 small
    # kernels remains).  So "auto" engages only for iterate() calls of >= graph_min_steps steps.
    graph = "auto"  # False disables
    graph_min_steps = 64

    def _graph_ok(self):
        v = self.system.value
        if self.graph is False or self.timing is not None or self.system.shard is not None:
            return False
        if self.path is not None or self.mcmc_queue or len(self.move_queue) != 1:
            return False
        if not getattr(self.move_queue[0], "graph_safe", False) or not hasattr(v, "graph_obs"):
            return False
        return all(getattr(r.eval, "fused_with", None) == self.move_queue[0].name for r in self.monitors.values())

    def _iterate_graph(self, n):
        sysm, v = self.system, self.system.value
        # The graph replays the steady state: after a step with resampling enabled the state
        # carries a deferred copy (v.pending) that the next move gathers.  A history read
        # materializes it (flush -> monitor -> data), and the very first call needs its
        # workspaces allocated: one eager step restores both before capture / replay.
        steady = (v.pending is not None) == (sysm.threshold > 0.0)
        if not getattr(self, "_graph_warm", False) or not steady:
            self._step()
            n -= 1
            self._graph_warm = True
        pairs = n // 2
        # never replay past the observations: the graph gathers obs[t] by a device index, so an
        # out-of-range t would be a device-side fault; the eager path raises IndexError instead
        nobs = v.obs.shape[0] if getattr(v, "obs", None) is not None else 0
        pairs = max(0, min(pairs, (nobs - 1 - self.iteration) // 2))
        if pairs == 0:
            return n
        # the captured moves advance the counter array itself: bring it up to date (an eager
        # move may have advanced the streams by a uniform count only) before capture / replay
        sysm.rng_set.counters
        t0 = self.iteration
        self._row(t0 + 2 * pairs)  # history capacity first: the graph bakes its address in
        ncols = len(self._cols)
        if getattr(self, "_gbuf", None) is None or self._gbuf["stage"].shape[1] != ncols:
            self._gbuf = {"stage": torch.zeros((2, ncols), dtype=torch.float64, device=self.device),
                          "t": torch.zeros(1, dtype=torch.int64, device=self.device),
                          "obs": torch.zeros((1, 2), dtype=torch.float64, device=self.device), "graphs": {}}
        gb = self._gbuf
        stage, tdev = gb["stage"], gb["t"]
        mon = {name: self._col[f"{name}.0"] for name in self.monitors}

        nobs_dev = v.obs.shape[0]

        def step(slot):
            prev = 1 - slot
            v.graph_obs = gb["obs"]  # this step's observation (gathered by the previous advance)
            accs = [apply_move(op, sysm, self.iteration + 1) for op in self.move_queue]
            # one launch: previous row (its monitor now fused in) -> history[t - 1], t += 1, the
            # next step's observation -> gb["obs"]
            _abi.call("smc_graph_advance", _abi.ptr(v.obs), nobs_dev, _abi.ptr(gb["obs"]),
                      ctypes.c_void_p(stage[prev].data_ptr()), _abi.ptr(self._hist), ncols, _abi.ptr(tdev),
                      _abi.stream())
            self._after_moves(self.iteration + 1, stage[slot], accs)

        # entry: the last eager row continues as the "previous" staging row
        stage[1].copy_(self._hist[t0])
        for name, col in mon.items():
            sysm.pending_monitors[name] = (stage[1].data_ptr() + 8 * col, t0)
        tdev.fill_(t0 + 1)
        gb["obs"].copy_(v.obs[t0 + 1:t0 + 2])  # the first replayed step's observation
        # everything the capture bakes in as a launch argument: buffers, and the sampler's public
        # knobs (threshold, scheme, RNG seed) -- a changed knob must not replay the old value
        key = (v._cur, v.pending is not None, self._hist.data_ptr(), v.obs.data_ptr(),
               sysm.weight_set.state.data_ptr(), float(sysm.threshold), int(sysm.resample_scheme),
               int(sysm.rng_set.seed), sysm.rng_set.counters.data_ptr(), v.obs.shape[0])
        g = gb["graphs"].get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # capture_begin/end directly: no gc pass, no cache flush
                g.capture_begin()
                step(0)
                step(1)
                g.capture_end()
            torch.cuda.current_stream().wait_stream(side)
            gb["graphs"][key] = g
            # the capture only recorded: state, weights and counters are untouched
            for name, col in mon.items():
                sysm.pending_monitors[name] = (stage[1].data_ptr() + 8 * col, t0)
        v.graph_obs = None
        for _ in range(pairs):
            g.replay()
        # exit: the last step's row (complete except its fused monitor) back into the history
        tl = t0 + 2 * pairs
        self._hist[tl].copy_(stage[1])
        for name, col in mon.items():
            sysm.pending_monitors[name] = (self._hist[tl].data_ptr() + 8 * col, tl)
        self.iteration = tl
        self._rows = max(self._rows, tl + 1)
        return n - 2 * pairs

    def _after_moves(self, t, row, accs):
        sysm = self.system
        ws = sysm.weight_set
        n = sysm.size
        hist_ptr = ctypes.c_void_p(row.data_ptr())
        # ESS trigger (F11: also after init)
        _abi.call("smc_ess_decide", ws.state_ptr, sysm.n_total, sysm.threshold, hist_ptr, _abi.stream())
        self._mark("resample", 0)
        if sysm.threshold > 0.0:
            gate = ws.field_ptr("resample")
            value = sysm.value
            if sysm.shard is not None:
                # global resample across the ranks: counts bit-identical to one GPU,
                # cross-rank surplus rows arrive in place, local pairs gathered by the next move
                value.materialize()
                rows = ctypes.c_void_p(value.raw.data_ptr())
                sysm.shard.resample(sysm, sysm.resample_scheme, gate, ws.field_ptr("status"), rows,
                                    8 * value.dim)
                value.pending = (sysm.parents, gate)
            elif getattr(value, "defer_copy", False):
                # parent map only; the next (gathering) move applies the copy
                value.materialize()
                sysm.resampler(sysm.resample_scheme, weight_set=ws, rng=sysm.rng_set, stream_index=n,
                               parents=sysm.parents, gate=gate, status=ws.field_ptr("status"))
                value.pending = (sysm.parents, gate)
            else:
                rows = getattr(value, "resample_rows", lambda: None)()
                sysm.resampler(sysm.resample_scheme, weight_set=ws, rng=sysm.rng_set, stream_index=n,
                               parents=sysm.parents, rows=rows[0] if rows else None,
                               row_bytes=rows[1] if rows else 0, gate=gate, status=ws.field_ptr("status"))
                if not rows:
                    value.copy_inplace(sysm.parents, gate)
            ws.set_equal_weight_if(gate, sysm.n_total)
        self._mark("resample", 1)
        mcmc = self.mcmc_queue if t > 0 else []  # initialize() runs no mcmc
        if mcmc and hasattr(sysm.value, "materialize"):
            sysm.value.materialize()  # mcmc kernels update the state in place
        for op in mcmc:
            accs.append(apply_move(op, sysm, t))
        for k, a in enumerate(accs):
            if isinstance(a, torch.Tensor):
                row[2 + k].copy_(a.reshape(()).to(torch.float64), non_blocking=True)
            elif a:
                row[2 + k].fill_(float(a))
        self._mark("monitor", 0)
        if self.path is not None:
            alpha, integrand, ld = apply_path_eval(self.path, sysm, t)
            self._path_grid.append(alpha)
            row[self._col["path.grid"]].fill_(alpha)
            self._reduce(integrand, ld, 1, row, self._col["path.integrand"])
        for name, rec in self.monitors.items():
            col = self._col[f"{name}.0"]
            fw = getattr(rec.eval, "fused_with", None)
            if fw and self.move_queue and self.move_queue[0].name == fw:
                # deferred: the next move reduces it from the state it loads (no extra pass);
                # flush() evaluates it here instead if the history is read first
                sysm.pending_monitors[name] = (row.data_ptr() + 8 * col, t)
                continue
            vals, ld = apply_monitor_eval(rec.eval, sysm, t, rec.dim)
            self._reduce(vals, ld, rec.dim, row, col)
        self._mark("monitor", 1)

    def flush(self):
        """Evaluate deferred monitors now (state and weights are unchanged since their step)."""
        sysm = self.system
        for name, (addr, t) in list(sysm.pending_monitors.items()):
            rec = self.monitors[name]
            vals, ld = apply_monitor_eval(rec.eval, sysm, t, rec.dim)
            self._reduce(vals, ld, rec.dim, self._hist[t], self._col[f"{name}.0"])
            del sysm.pending_monitors[name]

    # Optional per-phase CUDA events (bench.py's live per-kernel timing):
    # set ``sampler.timing = {}``; each phase gets a list of (start, end) events.
    timing = None

    def _mark(self, phase, edge):
        if self.timing is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        lst = self.timing.setdefault(phase, [])
        if edge == 0:
            lst.append([ev, None])
        else:
            lst[-1][1] = ev

    def _reduce(self, vals, ld, m, row, col):
        ws = self.system.weight_set
        n = self.system.size
        buf, nb = self._ws.get(_abi.lib().smc_weighted_reduce_workspace_bytes(n, m))
        shard = self.system.shard
        if shard is None:
            out = ctypes.c_void_p(row.data_ptr() + 8 * col)
            _abi.call("smc_weighted_reduce", _abi.ptr(vals), ld, m, _abi.ptr(ws.lw_raw), ws.state_ptr, n, out, buf,
                      nb, _abi.stream())
            return
        # shard: local weighted sums, allgathered and added in rank order (deterministic)
        loc = torch.empty(m, dtype=torch.float64, device=self.device)
        _abi.call("smc_weighted_reduce", _abi.ptr(vals), ld, m, _abi.ptr(ws.lw_raw), ws.state_ptr, n,
                  _abi.ptr(loc), buf, nb, _abi.stream())
        allp = shard.comm.allgather(loc)
        acc = allp[0].clone()
        for g in range(1, shard.world):
            acc += allp[g]
        row[col:col + m].copy_(acc)

    def check(self):
        """Synchronize and raise any device-side failure (SPEC.md:315 'propagates')."""
        self.system.weight_set.raise_if_failed()

    # -- results ---------------------------------------
    def history(self):
        self.flush()
        h = self._hist[: self._rows].cpu().numpy()
        d = {"iter": np.arange(self._rows)}
        for c, k in self._col.items():
            d[c] = h[:, k].copy()
        return d

    def history_array(self):
        self.flush()
        return self._hist[: self._rows].cpu().numpy()

    def history_row(self, t):
        """Device view of row t (after flushing deferred monitors)."""
        self.flush()
        return self._hist[t]

    def monitor_estimate(self, name, t):
        self.flush()
        rec = self.monitors[name]
        if not 0 <= t < self._rows:
            raise IndexError("iteration not recorded")
        k = self._col[f"{name}.0"]
        return self._hist[t, k:k + rec.dim].cpu().numpy()

    def path_log_zconst(self):
        if self.path is None:
            raise RuntimeError("no path sampling evaluator")
        h = self.history()
        return PathAccumulator(h["path.grid"], h["path.integrand"]).log_zconst

    @property
    def log_zconst(self):
        return self.system.weight_set.log_zconst

    def write_tsv(self, path_or_file, header_comments=()):
        """History as TSV (SPEC.md:369, 17 significant digits SPEC.md:653)."""
        h = self.history()
        cols = ["iter"] + self._cols
        lines = [f"# {c}" for c in header_comments]
        lines.append("\t".join(cols))
        for t in range(self._rows):
            vals = []
            for c in cols:
                v = h[c][t]
                if c in ("iter", "resampled") or c.startswith("accept."):
                    vals.append(str(int(round(v))))
                else:
                    vals.append(f"{v:.17g}")
            lines.append("\t".join(vals))
        text = "\n".join(lines) + "\n"
        if hasattr(path_or_file, "write"):
            path_or_file.write(text)
        else:
            with open(path_or_file, "w") as f:
                f.write(text)
        return text
