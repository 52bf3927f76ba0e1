"""Counter-based random streams on the device (mirror of smckit.rng, rng.py:1-215).

Same streams, same numbers: stream ``i`` of ``RngStreamSet(size, seed)`` is
Philox4x32-10 keyed by the seed, counter (draw_lo, draw_hi, i_lo, i_hi)
(rng.py:59-82).  Uniforms are bit-identical to the reference; normals and
gammas use the same algorithms (rng.py:85-117) with CUDA libdevice
transcendentals, so they agree with glibc to a few ulp.

The per-stream draw counters live in device memory (``counters``, uint64
stored as int64), so particle kernels advance them without host traffic.
``RngStream`` draws run as kernels; scalar draws synchronize to return a
Python float, vector draws return CUDA tensors.
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi

__all__ = ["RngStreamSet", "RngStream", "DRAW_U01", "DRAW_NORMAL", "DRAW_GAMMA"]

DRAW_U01, DRAW_NORMAL, DRAW_GAMMA = 0, 1, 2


class RngStreamSet:
    """``size`` independent streams keyed by a 64-bit seed (rng.py:138-170).

    A particle system of size N uses N + 1 streams: one per particle and the
    sampler-global (resampling) stream at index N (rng.py:3-5).
    """

    def __init__(self, size, seed=0, device="cuda"):
        size = int(size)
        if size < 1:
            raise ValueError(f"stream set needs at least one stream, got size={size}")
        seed = int(seed) % (1 << 64)
        _abi.require_cuda()
        self.size = size
        self.seed = seed
        self._k0 = seed & 0xFFFFFFFF
        self._k1 = seed >> 32
        self.device = torch.device(device)
        self.counters = torch.zeros(size, dtype=torch.int64, device=self.device)  # uint64 bit pattern

    @property
    def key(self):
        """Philox key words (low, high) derived from the master seed (rng.py:161-164)."""
        return self._k0, self._k1

    def stream(self, i) -> "RngStream":
        i = int(i)
        if not 0 <= i < self.size:
            raise IndexError(f"stream index {i} out of range [0, {self.size})")
        return RngStream(self, i)

    def counters_host(self):
        """Counter values as Python ints (uint64)."""
        return [int(c) & 0xFFFFFFFFFFFFFFFF for c in self.counters.cpu().tolist()]

    def counter_ptr(self, i):
        """Device address of stream i's counter (the resampling kernels advance it in place)."""
        return ctypes.c_void_p(self.counters.data_ptr() + 8 * int(i))

    def draw_streams(self, kind, first, n, shape=1.0, mean=0.0, scale=1.0, out=None):
        """One draw from each of streams first..first+n-1 (the per-particle pattern)."""
        first, n = int(first), int(n)
        if first < 0 or first + n > self.size:
            raise IndexError("stream range out of bounds")
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
        _abi.call("smc_rng_draw_streams", int(kind), self.seed, first, n, _abi.ptr(self.counters), float(shape),
                  float(mean), float(scale), _abi.ptr(out), _abi.stream())
        return out


class RngStream:
    """Handle on one stream (rng.py:173-215).  One user at a time per stream."""

    __slots__ = ("_set", "index")

    def __init__(self, stream_set, index):
        self._set = stream_set
        self.index = index

    def _fill(self, kind, n, shape, mean, scale):
        s = self._set
        m = 1 if n is None else int(n)
        out = torch.empty(m, dtype=torch.float64, device=s.device)
        _abi.call("smc_rng_fill", kind, s.seed, self.index, _abi.ptr(s.counters), float(shape), float(mean),
                  float(scale), _abi.ptr(out), m, _abi.stream())
        return float(out.item()) if n is None else out

    def uniform01(self, n=None):
        """Uniform draw(s) in [0, 1) -- bit-identical to rng.py:75-82."""
        return self._fill(DRAW_U01, n, 1.0, 0.0, 1.0)

    def normal(self, mean=0.0, sd=1.0, n=None):
        """mean + sd * z, z Box-Muller (rng.py:195-204)."""
        if not sd > 0.0:
            raise ValueError(f"normal needs sd > 0, got sd={sd}")
        return self._fill(DRAW_NORMAL, n, 1.0, mean, sd)

    def gamma(self, shape, scale=1.0, n=None):
        """scale * Gamma(shape) by Marsaglia-Tsang (rng.py:206-215)."""
        if not (shape > 0.0 and scale > 0.0):
            raise ValueError(f"gamma needs shape > 0 and scale > 0, got shape={shape}, scale={scale}")
        return self._fill(DRAW_GAMMA, n, shape, 0.0, scale)
