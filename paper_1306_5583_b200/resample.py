"""Resampling on the device (mirror of smckit.resample).

All six schemes share the pinned integer CDF contract of DESIGN.md (SURVEY.md
Appendix A), so the counts and the parent map are bit-identical to the CPU
oracle for identical normalized weights and uniforms, for any N and any
tiling.  Uniforms come from the sampler-global stream (index N) of the
supplied RngStreamSet, advanced on the device by the scheme's
draw count (multinomial/stratified: N, systematic: 1, residual variants: R).
"""

from __future__ import annotations

import ctypes
import enum

import torch

from . import _abi

__all__ = [
    "ResampleScheme", "resample", "resample_multinomial", "resample_stratified", "resample_systematic",
    "resample_residual", "resample_residual_stratified", "resample_residual_systematic",
    "replication_to_parents", "Resampler",
]


class ResampleScheme(enum.IntEnum):
    """SPEC.md:127-130 (closed set of four) + the two residual variants the north star adds."""

    Multinomial = 0
    Residual = 1
    Stratified = 2
    Systematic = 3
    ResidualStratified = 4
    ResidualSystematic = 5


def _scheme(s):
    if isinstance(s, str):
        key = s.replace("_", "").replace("-", "").lower()
        for m in ResampleScheme:
            if m.name.lower() == key:
                return m
        raise ValueError(f"unknown resampling scheme {s!r}")
    return ResampleScheme(int(s))


class Resampler:
    """Reusable device workspace + launch wrapper for ``smc_resample``."""

    def __init__(self, size, device="cuda"):
        self.size = int(size)
        self.device = torch.device(device)
        self._ws = _abi.Workspace(self.device)
        self.status = torch.zeros(3, dtype=torch.int32, device=self.device)  # smc_status

    def __call__(self, scheme, *, weights=None, weight_set=None, rng=None, stream_index=None, u=None,
                 m_out=None, counts=None, parents=None, rows=None, row_bytes=0, gate=None, status=None):
        n = self.size
        scheme = _scheme(scheme)
        m_out = n if m_out is None else int(m_out)
        w = None if weights is None else torch.as_tensor(weights, dtype=torch.float64, device=self.device).contiguous()
        if w is not None and w.numel() != n:
            raise ValueError("weights length != size")
        lw = st = None
        if w is None:
            if weight_set is None:
                raise ValueError("need weights or a weight_set")
            lw, st = _abi.ptr(weight_set.lw_raw), weight_set.state_ptr
        if u is not None:
            u = torch.as_tensor(u, dtype=torch.float64, device=self.device).contiguous()
            ctr, seed, sidx, n_u = None, 0, 0, u.numel()
        else:
            if rng is None:
                raise ValueError("need uniforms or an RngStreamSet")
            sidx = n if stream_index is None else int(stream_index)
            ctr, seed, n_u = rng.counter_ptr(sidx), rng.seed, 0
        ws, nb = self._ws.get(_abi.lib().smc_resample_workspace_bytes(n))
        _abi.call("smc_resample", int(scheme), _abi.ptr(w), lw, st, n, m_out, seed, sidx, ctr, _abi.ptr(u), n_u,
                  _abi.ptr(counts), _abi.ptr(parents), rows, int(row_bytes), gate,
                  status if status is not None else ctypes.c_void_p(self.status.data_ptr()), ws, nb, _abi.stream())

    def check(self):
        code, _, first = (int(v) for v in self.status.cpu().tolist())
        if code:
            self.status.zero_()
            raise _abi.SmcError(code, "device-side resampling failure", _abi.decode_index(first))


_resamplers = {}


def _get(n, device):
    key = (int(n), str(device))
    r = _resamplers.get(key)
    if r is None:
        r = _resamplers[key] = Resampler(n, device)
    return r


def resample(scheme, weights, rng=None, u=None, m_out=None, stream_index=None):
    """counts[N] (int32, CUDA) for normalized ``weights``.

    ``rng`` is an RngStreamSet; its stream ``stream_index`` (default N, the
    sampler-global stream) supplies the uniforms, or pass explicit ``u``.
    """
    w = torch.as_tensor(weights, dtype=torch.float64)
    dev = w.device if w.is_cuda else (rng.device if rng is not None else torch.device("cuda"))
    n = w.numel()
    r = _get(n, dev)
    counts = torch.empty(n, dtype=torch.int32, device=dev)
    if rng is not None and stream_index is None:
        stream_index = rng.size - 1
    r(scheme, weights=w.to(dev), rng=rng, stream_index=stream_index, u=u, m_out=m_out, counts=counts)
    r.check()
    return counts


def resample_multinomial(weights, rng=None, u=None):
    return resample(ResampleScheme.Multinomial, weights, rng, u)


def resample_stratified(weights, rng=None, u=None):
    return resample(ResampleScheme.Stratified, weights, rng, u)


def resample_systematic(weights, rng=None, u=None):
    return resample(ResampleScheme.Systematic, weights, rng, u)


def resample_residual(weights, rng=None, u=None, m_out=None):
    return resample(ResampleScheme.Residual, weights, rng, u, m_out)


def resample_residual_stratified(weights, rng=None, u=None):
    return resample(ResampleScheme.ResidualStratified, weights, rng, u)


def resample_residual_systematic(weights, rng=None, u=None):
    return resample(ResampleScheme.ResidualSystematic, weights, rng, u)


def replication_to_parents(counts):
    """copy_from[N] from counts: survivors keep their slot,
    zero-count slots take surplus children in ascending order."""
    c = torch.as_tensor(counts, dtype=torch.int32)
    dev = c.device if c.is_cuda else torch.device("cuda")
    c = c.to(dev).contiguous()
    n = c.numel()
    r = _get(n, dev)
    parents = torch.empty(n, dtype=torch.int32, device=dev)
    ws, nb = r._ws.get(_abi.lib().smc_resample_workspace_bytes(n))
    _abi.call("smc_replication_to_parents", _abi.ptr(c), n, _abi.ptr(parents),
              ctypes.c_void_p(r.status.data_ptr()), ws, nb, _abi.stream())
    r.check()
    return parents
