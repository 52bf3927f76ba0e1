"""WeightSet on the device (mirror of smckit.weights).

The set owns ``lw_raw`` (N doubles) and a device ``smc_wstate`` record; the
normalized log-weight is ``lw_raw - lse`` (or ``-log N`` after
``set_equal_weight``, which only flips a device flag).  Every mutation is one
fused kernel pass plus a one-block finalize that recomputes lse and ESS
("ESS is recomputed eagerly").  Mutations are collective only
(SPEC.md:93).  Errors (all -inf, NaN) are detected on the device; the eager
methods below check them and raise ``SmcError`` ("rejection with a
diagnostic"); the sampler's hot loop defers the check to its next sync.
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi

__all__ = ["WeightSet", "SET_LOG", "ADD_LOG", "SET_LIN", "MUL_LIN", "EQUAL"]

SET_LOG, ADD_LOG, SET_LIN, MUL_LIN, EQUAL = range(5)


class WeightSet:
    def __init__(self, size, device="cuda", check=True):
        size = int(size)
        if size < 1:
            raise ValueError("WeightSet needs size >= 1")
        _abi.require_cuda()
        self.size = size
        self.device = torch.device(device)
        self.check_eager = check
        self.lw_raw = torch.zeros(size, dtype=torch.float64, device=self.device)
        self.state = torch.zeros(_abi.WSTATE_BYTES, dtype=torch.uint8, device=self.device)
        self._ws = _abi.Workspace(self.device)
        self.set_equal_weight()

    # -- raw device handles --------------------------------------------------
    @property
    def state_ptr(self):
        return ctypes.c_void_p(self.state.data_ptr())

    def field_ptr(self, name):
        return ctypes.c_void_p(self.state.data_ptr() + _abi.WSTATE_OFF[name])

    def host_state(self) -> _abi.SmcWState:
        """Synchronizing snapshot of the device record."""
        raw = bytes(self.state.cpu().numpy().tobytes())
        return _abi.SmcWState.from_buffer_copy(raw)

    def raise_if_failed(self):
        st = self.host_state()
        if st.status != 0:
            code, idx = st.status, _abi.decode_index(st.err_index)
            self.clear_status()
            raise _abi.SmcError(code, "device-side weight failure", idx)

    def reset_log_zconst(self):
        """NormalizingConstant::initialize: log Z accumulator back to 0."""
        off = _abi.WSTATE_OFF["log_zconst"]
        self.state[off:off + 8].zero_()

    def clear_status(self):
        for f in ("status", "err_index"):
            off = _abi.WSTATE_OFF[f]
            self.state[off:off + 4].zero_()

    # -- collective mutations --------------------------------
    def _update(self, mode, values, accumulate_nc=False, check=None):
        v = None
        if values is not None:
            v = torch.as_tensor(values, dtype=torch.float64, device=self.device).contiguous()
            if v.numel() != self.size:
                raise ValueError(f"expected {self.size} values, got {v.numel()}")
        ws, nb = self._ws.get(_abi.lib().smc_weights_workspace_bytes(self.size))
        _abi.call("smc_weights_update", mode, _abi.ptr(self.lw_raw), _abi.ptr(v), self.size, self.state_ptr,
                  int(bool(accumulate_nc)), ws, nb, _abi.stream())
        if self.check_eager if check is None else check:
            self.raise_if_failed()

    def set_equal_weight(self):
        """weight = 1/N, ess = N."""
        self._update(EQUAL, None, check=False)

    def set_equal_weight_if(self, gate_ptr, n_total=None):
        """Device-gated set_equal_weight (the post-resample reset; no host sync).
        n_total: the global particle count of a sharded system (equal weight 1/n_total)."""
        _abi.call("smc_weights_set_equal", self.state_ptr, int(n_total or self.size), gate_ptr, _abi.stream())

    def set_log_weight(self, values, accumulate_nc=False, check=None):
        """Normalize values by max-shift + log-sum-exp.  accumulate_nc:
        log_zconst += log mean exp(values) (the initial weights' contribution to log Z)."""
        self._update(SET_LOG, values, accumulate_nc, check=check)

    def add_log_weight(self, increments, accumulate_nc=False, check=None):
        """log_weight += increments, renormalize."""
        self._update(ADD_LOG, increments, accumulate_nc, check=check)

    def set_weight(self, values, check=None):
        """Linear-domain set."""
        self._update(SET_LIN, values, check=check)

    def mul_weight(self, factors, check=None):
        """Linear-domain multiply."""
        self._update(MUL_LIN, factors, check=check)

    # -- reads ----------------------------------------------------------------
    def ess(self):
        """1 / sum_i W_i^2; synchronizes."""
        return self.host_state().ess

    def read_weight(self):
        """Snapshot copy of the normalized weights."""
        out = torch.empty(self.size, dtype=torch.float64, device=self.device)
        _abi.call("smc_weights_read", 1, _abi.ptr(self.lw_raw), self.state_ptr, self.size, _abi.ptr(out),
                  _abi.stream())
        return out

    def read_log_weight(self):
        out = torch.empty(self.size, dtype=torch.float64, device=self.device)
        _abi.call("smc_weights_read", 0, _abi.ptr(self.lw_raw), self.state_ptr, self.size, _abi.ptr(out),
                  _abi.stream())
        return out

    @property
    def log_zconst(self):
        return self.host_state().log_zconst
