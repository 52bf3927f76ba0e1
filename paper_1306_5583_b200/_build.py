"""Build the sm_100a shared library (libsmcb200.so) in-tree with nvcc.

The library is the product: every kernel of the SMC hot path plus the C ABI of
include/smc_abi.h.  It is compiled for sm_100a only (no PTX fallback, no other
architectures) with --fmad=false so the fp64 arithmetic rounds exactly as the
reference's numba code (no FMA contraction).
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("SMC_LIB_PATH") or os.path.join(HERE, "libsmcb200.so")  # override: A/B experiments

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-diag-suppress", "20091",  # host-side instantiation of the fast-math tables (host tests use their own build)
]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    """Every file the library is compiled from: kernels, device headers, the fast-math tables."""
    pats = ("*.cu", "*.cuh", "*.h", "*.inc")
    files = [f for p in pats for f in glob.glob(os.path.join(CSRC, p))]
    return sorted(files + glob.glob(os.path.join(ROOT, "include", "*.h")))


def source_hash():
    """sha256 over the build flags and every source file (the library's stamp)."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for f in _deps():
        h.update(os.path.relpath(f, ROOT).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


STAMP = LIB + ".stamp"


def _stale():
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            return f.read().strip() != source_hash()
    except OSError:
        return True


def build(force=False, verbose=False, extra=()):
    """Compile csrc/*.cu into paper_1306_5583_b200/libsmcb200.so (sm_100a)."""
    if not force and not _stale():
        return LIB
    if not force and os.environ.get("SMC_LIB_PATH") and os.path.exists(LIB):
        return LIB  # an A/B variant is used as built, never rebuilt from the current sources
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *sources()]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout, r.stderr, file=sys.stderr)
    os.replace(LIB + ".tmp", LIB)
    if not extra:
        with open(STAMP, "w") as f:
            f.write(source_hash())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=("-Xptxas", "-v") if "--ptxas-v" in sys.argv else ())
    print(LIB)
