"""The C-ABI library loads and exports every symbol include/smc_abi.h declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_1306_5583_b200 import _abi, _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "smc_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t)\s+(smc_\w+)\s*\(", src, flags=re.M)))


def test_library_built_for_sm100a():
    path = _build.build()
    assert os.path.exists(path)
    assert "arch=compute_100a,code=sm_100a" in " ".join(_build.NVCC_FLAGS)


def test_exports_every_header_symbol():
    lib = ctypes.CDLL(_abi.library_path())
    names = header_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_abi.EXPORTS), set(names) ^ set(_abi.EXPORTS)


def test_host_only_entry_points():
    lib = _abi.load()
    assert lib.smc_abi_version() == 3
    assert lib.smc_resample_workspace_bytes(1 << 20) > (1 << 20) * 20
    assert lib.smc_weights_workspace_bytes(1000) > 0
    assert lib.smc_pf_workspace_bytes(1000) > 0
    assert lib.smc_weighted_reduce_workspace_bytes(1000, 2) > 0
    # a production build: no index guards compiled in, nothing to report (no CUDA call made)
    assert _abi.check_failures() == (False, 0, "")


def test_argument_validation_without_gpu():
    lib = _abi.load()
    # bad scheme / null pointers are rejected on the host before any launch
    rc = lib.smc_resample(9, None, None, None, 10, 10, 0, 10, None, None, 0, None, None, None, 0, None, None,
                          None, 0, None)
    assert rc == -1
    assert "bad scheme" in _abi.last_error()
    rc = lib.smc_weights_update(0, None, None, 0, None, 0, None, 0, None)
    assert rc == -1
    with pytest.raises(_abi.SmcError):
        _abi.check(-7)


def test_wstate_layout_matches_header():
    assert _abi.WSTATE_BYTES == 88
    assert _abi.WSTATE_OFF["status"] == 68 and _abi.WSTATE_OFF["resample"] == 72
    # the smc_status convention: the first failing index sits 8 bytes after the status word
    assert _abi.WSTATE_OFF["err_index"] == _abi.WSTATE_OFF["status"] + 8
    assert _abi.decode_index(0) is None and _abi.decode_index(0x7FFFFFFF - 123) == 123
