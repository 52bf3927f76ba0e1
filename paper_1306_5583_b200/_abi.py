"""ctypes binding of include/smc_abi.h (the drop-in C ABI).

The product path has no CPU fallback: if libsmcb200.so is missing it is built
with nvcc (sm_100a), and if that fails or no CUDA device is present every
call raises.  Device buffers are torch CUDA tensors; the stream of every call
is torch's current stream.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from . import _build

_lib = None
_lock = threading.Lock()

SMC_OK = 0
ERRORS = {
    -1: "invalid argument",
    -2: "unnormalized resampling input (SPEC.md:137)",
    -3: "weight normalization failure: all -inf / NaN (SPEC.md:45)",
    -4: "not enough uniforms for the scheme",
    -5: "replication counts do not sum to N (SPEC.md:169)",
    -6: "CUDA error",
    -7: "workspace too small",
}


class SmcError(RuntimeError):
    """Raised for every failure the ABI reports (host- or device-detected).  ``index`` is the
    first (lowest-index) failing particle when the device named one."""

    def __init__(self, code, msg="", index=None):
        self.code = code
        self.index = index
        where = f" (first failing particle {index})" if index is not None else ""
        super().__init__(f"[{code}] {ERRORS.get(code, 'error')}{': ' + msg if msg else ''}{where}")


def decode_index(v):
    """smc_status.first_index (INT32_MAX - index, 0 = none) -> index or None."""
    v = int(v)
    return None if v <= 0 else 0x7FFFFFFF - v


class SmcWState(C.Structure):
    """Mirror of smc_wstate (include/smc_abi.h)."""

    _fields_ = [
        ("lse", C.c_double), ("ess", C.c_double), ("ess_over_n", C.c_double), ("nc_inc", C.c_double),
        ("log_zconst", C.c_double), ("max_raw", C.c_double), ("log_sum", C.c_double), ("w_equal", C.c_double),
        ("equal", C.c_int32), ("status", C.c_int32),
        ("resample", C.c_int32), ("err_index", C.c_int32),
        ("lse_ticket", C.c_uint32), ("reserved", C.c_uint32),
    ]


WSTATE_BYTES = C.sizeof(SmcWState)
WSTATE_OFF = {name: getattr(SmcWState, name).offset for name, _ in SmcWState._fields_}

_vp, _i64, _u64, _i32, _f64, _sz = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_size_t

_SIGS = {
    "smc_abi_version": ([], C.c_int),
    "smc_last_error": ([C.c_char_p, _sz], C.c_int),
    "smc_launch_count": ([_vp], C.c_int),
    "smc_check_failures": ([_vp, _vp, C.c_char_p, _sz], C.c_int),
    "smc_graph_advance": ([_vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp], C.c_int),
    "smc_philox_blocks": ([_vp, _i64, _u64, _vp, _vp], C.c_int),
    "smc_rng_fill": ([_i32, _u64, _u64, _vp, _f64, _f64, _f64, _vp, _i64, _vp], C.c_int),
    "smc_rng_draw_streams": ([_i32, _u64, _u64, _i64, _vp, _f64, _f64, _f64, _vp, _vp], C.c_int),
    "smc_weights_workspace_bytes": ([_i64], _sz),
    "smc_weights_update": ([_i32, _vp, _vp, _i64, _vp, _i32, _vp, _sz, _vp], C.c_int),
    "smc_weights_set_equal": ([_vp, _i64, _vp, _vp], C.c_int),
    "smc_weights_read": ([_i32, _vp, _vp, _i64, _vp, _vp], C.c_int),
    "smc_ess_decide": ([_vp, _i64, _f64, _vp, _vp], C.c_int),
    "smc_weighted_reduce_workspace_bytes": ([_i64, _i64], _sz),
    "smc_weighted_reduce": ([_vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp], C.c_int),
    "smc_resample_workspace_bytes": ([_i64], _sz),
    "smc_resample": ([_i32, _vp, _vp, _vp, _i64, _i64, _u64, _u64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                      _vp, _vp, _sz, _vp], C.c_int),
    "smc_debug_set": ([C.c_int, C.c_int], C.c_int),
    "smc_weights_combine": ([_vp, _i32, _vp, _i64, _i32, _i32, _vp, _vp], C.c_int),
    "smc_resample_shard_totals": ([_i32, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _sz, _vp, _vp],
                                  C.c_int),
    "smc_resample_shard_counts": ([_i32, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _vp, _u64, _u64, _vp, _vp,
                                   _i64, _vp, _vp, _vp, _vp, _sz, _vp, _vp], C.c_int),
    "smc_resample_shard_pack": ([_vp, _i64, _i64, _vp, _i32, _vp, _vp, _sz, _vp], C.c_int),
    "smc_resample_shard_assign": ([_vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp], C.c_int),
    "smc_resample_shard_assign_p2p": ([_vp, _i32, _i32, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "smc_replication_to_parents": ([_vp, _i64, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "smc_gather_rows": ([_vp, _vp, _i64, _vp, _i64, _vp], C.c_int),
    "smc_copy_rows_inplace": ([_vp, _i64, _vp, _i64, _vp, _vp], C.c_int),
    "smc_gmm_init": ([_vp, _i64, _i32, _u64, _u64, _vp, _vp, _i32, _vp, _vp], C.c_int),
    "smc_gmm_eval": ([_vp, _i64, _i32, _vp, _i32, _vp, _vp], C.c_int),
    "smc_gmm_workspace_bytes": ([_i64], _sz),
    "smc_gmm_reweight": ([_vp, _vp, _i64, _f64, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "smc_gmm_mh": ([_i32, _vp, _i64, _i32, _u64, _u64, _vp, _vp, _i32, _vp, _f64, _f64, _vp, _vp], C.c_int),
    "smc_user_compile": ([C.c_char_p, _vp, _i32, _vp, C.c_char_p, _sz], C.c_int),
    "smc_user_kind": ([_vp], C.c_int),
    "smc_user_free": ([_vp], C.c_int),
    "smc_user_launch_move": ([_vp, _u64, _vp, _i64, _i32, _i32, _u64, _u64, _vp, _vp, _i32, _vp, _vp, _vp], C.c_int),
    "smc_user_launch_eval": ([_vp, _u64, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp], C.c_int),
    "smc_pf_workspace_bytes": ([_i64], _sz),
    "smc_pf_init": ([_vp, _vp, _i64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "smc_pf_move": ([_vp, _vp, _vp, _vp, _vp, _i64, _u64, _i64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
                    C.c_int),
    "smc_pf_move_uniform": ([_vp, _vp, _vp, _vp, _vp, _i64, _u64, _i64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp,
                             _sz, _vp], C.c_int),
}
EXPORTS = tuple(_SIGS)


def library_path():
    return _build.LIB


def load(build_if_missing=True):
    """Load libsmcb200.so (building it in-tree if needed); no GPU required."""
    global _lib
    with _lock:
        if _lib is None:
            if build_if_missing:
                _build.build()
            if not os.path.exists(_build.LIB):
                raise ImportError(f"{_build.LIB} is missing: the CUDA library is required (no CPU fallback)")
            L = C.CDLL(_build.LIB)
            for name, (args, res) in _SIGS.items():
                if os.environ.get("SMC_LIB_PATH") and not hasattr(L, name):
                    continue  # an older A/B variant without a newer entry point
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            _lib = L
    return _lib


def lib():
    return _lib if _lib is not None else load()


def launch_count():
    """Kernels the library has launched in this process (smc_launch_count)."""
    v = C.c_uint64(0)
    lib().smc_launch_count(C.byref(v))
    return int(v.value)


def check_failures():
    """(checked_build, violated index guards, 'file:line' of the first) -- smc_check_failures."""
    f, ln = C.c_uint64(0), C.c_uint64(0)
    buf = C.create_string_buffer(256)
    checked = lib().smc_check_failures(C.byref(f), C.byref(ln), buf, 256)
    where = f"{buf.value.decode(errors='replace')}:{ln.value}" if f.value else ""
    return bool(checked), int(f.value), where


def last_error():
    buf = C.create_string_buffer(512)
    lib().smc_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc):
    if rc != SMC_OK:
        raise SmcError(rc, last_error())


def require_cuda():
    if not torch.cuda.is_available():
        raise SmcError(-6, "no CUDA device: the B200 path has no CPU fallback")


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Raw device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise SmcError(-1, "tensor must live on the CUDA device")
    if not t.is_contiguous():
        raise SmcError(-1, "tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def call(name, *args):
    check(getattr(lib(), name)(*args))


class Workspace:
    """Grow-only device scratch (the library never allocates)."""

    def __init__(self, device):
        self.device = device
        self.buf = None

    def get(self, nbytes):
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            if os.environ.get("SMC_CHECKED_RUN"):  # checked runs: no reliance on zeroed scratch
                self.buf.fill_(0xA5)
        return C.c_void_p(self.buf.data_ptr()), C.c_size_t(self.buf.numel())
