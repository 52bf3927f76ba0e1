"""Counter-based random streams on the device (mirror of smckit.rng, rng.py:1-215).

Same streams, same numbers: stream ``i`` of ``RngStreamSet(size, seed)`` is
Philox4x32-10 keyed by the seed, counter (draw_lo, draw_hi, i_lo, i_hi)
(rng.py:59-82).  Uniforms are bit-identical to the reference; normals and
gammas use the same algorithms (rng.py:85-117) with the branch-free fp64
pieces of smc_fastmath.h (table log, cos_bm, sqrt_bm; libdevice pow for the
gamma boost), so they agree with glibc to a few ulp.

The per-stream draw counters live in device memory (``counters``, uint64
stored as int64), so particle kernels advance them without host traffic.
``RngStream`` draws run as kernels; scalar draws synchronize to return a
Python float, vector draws return CUDA tensors.
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi

__all__ = ["RngStreamSet", "RngStream", "DRAW_U01", "DRAW_NORMAL", "DRAW_GAMMA", "philox_block", "u01",
           "std_normal", "std_gamma", "fill_u01", "fill_std_normal", "fill_std_gamma", "sample_uniform01",
           "sample_normal", "sample_gamma"]

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
        self._ctr = torch.zeros(size, dtype=torch.int64, device=self.device)  # uint64 bit pattern
        # Uniform-count knowledge: streams [0, _u_n) all sit at draw count _u_val; when
        # _u_stale the device array lags (a uniform-counter move advanced them without
        # writing it) and is brought up to date before anyone else sees it.
        self._u_n, self._u_val, self._u_stale = size, 0, False

    @property
    def counters(self):
        """The device counter array (up to date).  The caller may change it, so the
        uniform-count knowledge is dropped."""
        self._materialize()
        self._u_n = 0
        return self._ctr

    def _materialize(self):
        if self._u_stale:
            if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
                raise RuntimeError("stream counters are lazily advanced: read them before a graph capture")
            v = self._u_val - (1 << 64) if self._u_val >= (1 << 63) else self._u_val
            self._ctr[:self._u_n].fill_(v)
            self._u_stale = False

    def uniform_count(self, n, draws):
        """The common draw count of streams [0, n) if known, and if ``draws`` more draws
        do not carry into the counter's high word (``draws`` = 0: no such check); else None."""
        if self._u_n < n or (draws and (self._u_val & 0xFFFFFFFF) > 0x100000000 - draws):
            return None
        if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
            return None  # a captured graph replays: the count must come from the array
        return self._u_val

    def advance_uniform(self, n, val, written):
        """Streams [0, n) now all sit at ``val``; ``written``: the array holds it too."""
        self._u_n, self._u_val = n, val
        self._u_stale = not written

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
        i = int(i)
        if i < self._u_n:  # streams [i, _u_n) leave the uniform prefix
            self._materialize()
            self._u_n = i
        return ctypes.c_void_p(self._ctr.data_ptr() + 8 * i)

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
        s.counter_ptr(self.index)  # stream `index` leaves the uniform prefix
        _abi.call("smc_rng_fill", kind, s.seed, self.index, _abi.ptr(s._ctr), float(shape), float(mean),
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


# -- the reference's compiled-kernel primitives (rng.py:59-135) on device counters -------------
# smckit calls these from numba kernels on a host counter array; here ``ctrs`` is the device
# counter tensor of an RngStreamSet (int64 holding the uint64 bits) and (k0, k1) the key
# halves, exactly as ``RngStreamSet.key`` returns them.  Scalar forms synchronize.
def philox_block(c0, c1, c2, c3, k0, k1):
    """One Philox4x32-10 block (rng.py:59-72) -> 4 uint32 words."""
    _abi.require_cuda()
    import numpy as np
    ctr = torch.tensor(np.array([c0, c1, c2, c3], np.uint32).view(np.int32), device="cuda")
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    _abi.call("smc_philox_blocks", _abi.ptr(ctr), 1, (int(k0) & 0xFFFFFFFF) | ((int(k1) & 0xFFFFFFFF) << 32),
              _abi.ptr(out), _abi.stream())
    return tuple(int(w) for w in out.cpu().numpy().view(np.uint32))


def _draw(kind, ctrs, i, k0, k1, shape, out):
    if not (isinstance(ctrs, torch.Tensor) and ctrs.is_cuda and ctrs.dtype == torch.int64):
        raise TypeError("ctrs must be the CUDA int64 counter tensor of an RngStreamSet")
    if not 0 <= int(i) < ctrs.numel():
        raise IndexError("stream index out of range")
    seed = (int(k0) & 0xFFFFFFFF) | ((int(k1) & 0xFFFFFFFF) << 32)
    _abi.call("smc_rng_fill", kind, seed, int(i), _abi.ptr(ctrs), float(shape), 0.0, 1.0, _abi.ptr(out),
              out.numel(), _abi.stream())
    return out


def u01(ctrs, i, k0, k1):
    """Uniform in [0, 1) from stream i, advancing ctrs[i] (rng.py:75-82); bit-exact."""
    return float(_draw(DRAW_U01, ctrs, i, k0, k1, 1.0, torch.empty(1, dtype=torch.float64, device=ctrs.device)))


def std_normal(ctrs, i, k0, k1):
    """Box-Muller normal, two draws (rng.py:85-91)."""
    return float(_draw(DRAW_NORMAL, ctrs, i, k0, k1, 1.0, torch.empty(1, dtype=torch.float64, device=ctrs.device)))


def std_gamma(ctrs, i, k0, k1, shape):
    """Marsaglia-Tsang gamma(shape, 1) (rng.py:94-117)."""
    if not shape > 0.0:
        raise ValueError("gamma needs shape > 0")
    return float(_draw(DRAW_GAMMA, ctrs, i, k0, k1, shape, torch.empty(1, dtype=torch.float64, device=ctrs.device)))


def fill_u01(ctrs, i, k0, k1, out):
    """out[:] = consecutive uniforms of stream i (rng.py:120-124); out is a CUDA float64 tensor."""
    return _draw(DRAW_U01, ctrs, i, k0, k1, 1.0, out)


def fill_std_normal(ctrs, i, k0, k1, out):
    return _draw(DRAW_NORMAL, ctrs, i, k0, k1, 1.0, out)


def fill_std_gamma(ctrs, i, k0, k1, shape, out):
    if not shape > 0.0:
        raise ValueError("gamma needs shape > 0")
    return _draw(DRAW_GAMMA, ctrs, i, k0, k1, shape, out)


# -- SPEC.md:221-223 operation names ---------------------------------------------------------
def sample_uniform01(stream):
    return stream.uniform01()


def sample_normal(stream, mean, sd):
    return stream.normal(mean, sd)


def sample_gamma(stream, shape, scale):
    return stream.gamma(shape, scale)
