"""User particle kernels compiled at run time (the generic plugin path).

The reference's user code is a per-particle function
``kernel(iter, SingleParticleView) -> int`` (C++
``move_state(iter, SingleParticle<T>)`` PAPER.md:866-871 via MoveAdapter
:944-982) plus monitor / path evaluators.  Here
the user writes that function in CUDA C++ against ``smc_user.cuh``; NVRTC
compiles it for sm_100a at run time (``smc_user_compile`` in the C ABI) and it
runs as one thread per particle with the same own-slot contract.  No Python
runs per particle, and there is no CPU path.

    src = r'''
    #include "smc_user.cuh"
    __device__ int rw_move(smc::Particle &p, unsigned long long iter, const double *prm)
    {
        double x = p.state(0) + p.normal(0.0, prm[0]);
        p.slot(0) = -0.5 * x * x;          // incremental log weight -> post
        p.state(0) = x;
        return 0;
    }
    SMC_USER_MOVE(rw_move)
    '''
    move = user.compile_move(src, scratch_dim=1, params=torch.tensor([0.5], device="cuda"),
                             post=user.add_scratch_log_weight(0))
    sampler.add_move(move)
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _abi
from .core import COL_MAJOR
from .exec import MonitorEval, ParticleKernelOp, PathEval

__all__ = ["UserKernel", "compile_move", "compile_monitor", "compile_path", "add_scratch_log_weight",
           "set_scratch_log_weight", "scratch", "INCLUDE_DIR"]

INCLUDE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
MOVE, EVAL = 1, 2


class UserKernel:
    """A compiled module holding one ``smc_user_entry`` kernel."""

    def __init__(self, source, options=()):
        _abi.require_cuda()
        opts = [f"-I{INCLUDE_DIR}", *options]
        arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
        handle = ctypes.c_void_p()
        log = ctypes.create_string_buffer(1 << 16)
        L = _abi.lib()
        rc = L.smc_user_compile(source.encode(), ctypes.cast(arr, ctypes.c_void_p), len(opts), ctypes.byref(handle),
                                log, len(log))
        self.log = log.value.decode(errors="replace")
        if rc != _abi.SMC_OK:
            raise _abi.SmcError(rc, _abi.last_error() + ("\n" + self.log if self.log else ""))
        self._h = handle
        self.kind = L.smc_user_kind(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _abi._lib is not None:
            _abi._lib.smc_user_free(h)
            self._h = None

    def launch_move(self, iter_, x, n, dim, col_major, stream_base, seed, ctrs, scratch_t, sdim, params, acc):
        _abi.call("smc_user_launch_move", self._h, int(iter_), _abi.ptr(x), n, dim, int(col_major),
                  int(stream_base), int(seed), _abi.ptr(ctrs), _abi.ptr(scratch_t), sdim, _abi.ptr(params),
                  _abi.ptr(acc), _abi.stream())

    def launch_eval(self, iter_, x, n, dim, col_major, params, out, m):
        _abi.call("smc_user_launch_eval", self._h, int(iter_), _abi.ptr(x), n, dim, int(col_major),
                  _abi.ptr(params), _abi.ptr(out), m, _abi.stream())


def scratch(system, cols):
    """The system's N x cols per-particle scratch (own slot only)."""
    s = getattr(system, "_user_scratch", None)
    if s is None or s.shape[1] < cols:
        s = system._user_scratch = torch.zeros((system.size, max(cols, 1)), dtype=torch.float64,
                                               device=system.device)
    return s


def _params(params, iter_, system):
    p = params(iter_, system) if callable(params) else params
    if p is None:
        return None
    if not (isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float64):
        raise TypeError("params must be a CUDA float64 tensor (or a callable returning one)")
    return p.contiguous()


def _state(system):
    v = system.value
    v.materialize()  # a deferred resample copy lands before user code reads rows
    return v.raw, v.dim, v.order == COL_MAJOR


def compile_move(source, scratch_dim=0, params=None, pre=None, post=None, name=None, options=()):
    """ParticleKernelOp whose kernel is the user's SMC_USER_MOVE function.
    params: CUDA f64 tensor or ``callable(iter, system) -> tensor`` handed to the kernel."""
    k = UserKernel(source, options)
    if k.kind != MOVE:
        raise ValueError("source defines an evaluator (SMC_USER_EVAL), not a move")

    def kernel(iter_, system):
        x, dim, col = _state(system)
        sc = scratch(system, scratch_dim) if scratch_dim else None
        acc = torch.zeros(1, dtype=torch.int64, device=system.device)
        k.launch_move(iter_, x, system.size, dim, col, system.stream_base, system.rng_set.seed,
                      system.rng_set.counters, sc, scratch_dim if sc is not None else 0,
                      _params(params, iter_, system), acc)
        return acc

    op = ParticleKernelOp(kernel, pre, post, name or "user_move")
    op.module = k
    return op


def _eval_kernel(source, options):
    k = UserKernel(source, options)
    if k.kind != EVAL:
        raise ValueError("source defines a move (SMC_USER_MOVE), not an evaluator")
    return k


def compile_monitor(source, dim, params=None, options=()):
    """MonitorEval from an SMC_USER_EVAL function writing out[0..dim) per particle."""
    k = _eval_kernel(source, options)

    def fn(iter_, system):
        x, d, col = _state(system)
        out = torch.empty(system.size * dim, dtype=torch.float64, device=system.device)
        k.launch_eval(iter_, x, system.size, d, col, _params(params, iter_, system), out, dim)
        return out, dim

    ev = MonitorEval(fn, dim)
    ev.module = k
    return ev


def compile_path(source, grid, params=None, options=()):
    """PathEval: integrand from an SMC_USER_EVAL function (out[0]); grid(iter, system) -> alpha_t."""
    k = _eval_kernel(source, options)

    def fn(iter_, system):
        x, d, col = _state(system)
        out = torch.empty(system.size, dtype=torch.float64, device=system.device)
        k.launch_eval(iter_, x, system.size, d, col, _params(params, iter_, system), out, 1)
        return float(grid(iter_, system)), out, 1

    ev = PathEval(fn)
    ev.module = k
    return ev


def set_scratch_log_weight(col=0, accumulate_nc=True):
    """A ``post`` hook for an init op: set_log_weight(scratch[:, col])."""

    def post(iter_, system):
        sc = scratch(system, col + 1)
        system.weight_set.set_log_weight(sc[:, col], accumulate_nc=accumulate_nc, check=False)

    return post


def add_scratch_log_weight(col=0, accumulate_nc=True):
    """A ``post`` hook: add_log_weight(scratch[:, col]) with the NC increment
    (nc_add_log_weight then add_log_weight) -- the usual end of a
    whole-system move."""

    def post(iter_, system):
        sc = scratch(system, col + 1)
        system.weight_set.add_log_weight(sc[:, col], accumulate_nc=accumulate_nc, check=False)

    return post
