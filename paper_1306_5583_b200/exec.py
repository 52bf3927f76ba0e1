"""Per-particle operation application (mirror of smckit.exec).

The reference applies ``kernel(iter, SingleParticleView) -> int`` to every
particle from a Sequential loop or a ThreadPool.  Here the
loop IS a CUDA grid: a particle kernel is a device launch covering all N
particles, one thread per particle, under the same own-slot contract
(write only your particle's state row, its RNG stream and
its scratch slot).  ``pre``/``post`` stay host callables run once per
application.  Acceptance counts are summed on the device in a
fixed order, so every result is independent of launch configuration -- the
GPU restatement of the backend-equivalence theorem.

There is no per-particle Python callback path: a kernel is a callable
``(iter, system) -> accept`` that launches device work (``accept`` is None,
an int, or a device int64 scalar).  Python per-particle callables would be a
CPU fallback, which this package does not have.
"""

from __future__ import annotations

import enum

import torch

__all__ = ["Backend", "ParticleKernelOp", "apply_move", "apply_monitor_eval", "apply_path_eval",
           "make_op_from_kernel", "MonitorEval", "PathEval"]


class Backend(enum.Enum):
    """SPEC.md:388-391.  The CUDA grid replaces Sequential/ThreadPool(k)."""

    CUDA = "cuda"


class ParticleKernelOp:
    """pre(iter, system) -> kernel(iter, system) [device, all particles] -> post(iter, system)."""

    def __init__(self, kernel, pre=None, post=None, name=None):
        if not callable(kernel):
            raise TypeError("kernel must be a callable launching device work")
        self.kernel = kernel
        self.pre = pre
        self.post = post
        self.name = name or getattr(kernel, "__name__", type(kernel).__name__)

    def __call__(self, iter_, system):
        return apply_move(self, system, iter_)


def make_op_from_kernel(kernel_fn, pre=None, post=None, name=None):
    """Adapter from plain functions to the op shape."""
    return ParticleKernelOp(kernel_fn, pre, post, name)


def apply_move(op, system, iter_, backend=Backend.CUDA):
    """pre, kernel over all particles, post; returns the summed acceptance count."""
    if backend is not Backend.CUDA:
        raise ValueError("only the CUDA backend exists")
    if op.pre is not None:
        op.pre(iter_, system)
    acc = op.kernel(iter_, system)
    if op.post is not None:
        op.post(iter_, system)
    return 0 if acc is None else acc


class MonitorEval:
    """Monitor evaluator: returns the N x m values as a device matrix view.

    ``fn(iter, system) -> (vals, ld)`` where ``vals`` is a CUDA float64 tensor
    whose row i starts at element i*ld and holds h_1..h_m(X_i)
    (res[i*dim + j]).  A view of the state matrix costs no copy.
    """

    def __init__(self, fn, dim):
        if int(dim) < 1:
            raise ValueError("monitor dimension must be >= 1 (SPEC.md:409)")
        self.fn = fn
        self.dim = int(dim)

    def __call__(self, iter_, system):
        return self.fn(iter_, system)


def apply_monitor_eval(ev, system, iter_, m=None):
    vals, ld = ev(iter_, system)
    if vals.dtype != torch.float64 or not vals.is_cuda:
        raise TypeError("monitor values must be a CUDA float64 tensor")
    return vals, int(ld)


class PathEval:
    """``fn(iter, system) -> (alpha_t, integrand[N] CUDA f64)``."""

    def __init__(self, fn):
        self.fn = fn

    def __call__(self, iter_, system):
        return self.fn(iter_, system)


def apply_path_eval(ev, system, iter_):
    """-> (alpha_t, vals, ld): integrand_i = vals[i * ld] (ld = 1 for a plain vector)."""
    r = ev(iter_, system)
    if len(r) == 3:
        return float(r[0]), r[1], int(r[2])
    return float(r[0]), r[1], 1
