"""Generate golden RNG vectors by importing the REFERENCE smckit.rng (rng.py:1-215).

Run here (the container that has /root/reference); the output is committed as
tests/golden/rng_golden.json so the GPU box (which has no /root/reference) can
check both the CPU oracle and the device kernels against the reference's own
draws.  Floats are stored with float.hex() so the comparison is bit-exact.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

(Both variables keep the import from writing __pycache__ into the read-only
reference tree.)
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from smckit import rng as R  # noqa: E402  (the reference module, unmodified)


def hx(a):
    return [float(v).hex() for v in np.atleast_1d(a)]


def main(out_path):
    g = {"source": "reference smckit.rng (pkg/src/smckit/rng.py)", "philox": [], "streams": [],
         "fills": [], "draw_sets": []}

    # Raw Philox4x32-10 blocks (rng.py:59-72), incl. the Random123 KAT vectors.
    blocks = [
        ((0, 0, 0, 0), (0, 0)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)),
        ((0, 0, 2, 0), (12345, 0)),
        ((1, 0, 2, 0), (12345, 0)),
        ((2, 0, 2, 0), (12345, 0)),
        ((7, 3, 0xDEADBEEF, 1), (0x9E3779B9, 77)),
    ]
    for ctr, key in blocks:
        c = tuple(np.uint64(v) for v in ctr)
        k = tuple(np.uint64(v) for v in key)
        out = R._philox_block(*c, *k)
        g["philox"].append({"ctr": list(ctr), "key": list(key), "out": [int(v) for v in out]})

    # Per-stream sequences through the public RngStream API (rng.py:173-215):
    # mixed u01 / normal / gamma calls, recording every value and the counter.
    cases = [
        (1306, 5, 0), (1306, 5, 1), (1306, 5, 2), (1306, 5, 3), (1306, 5, 4),
        (0, 1, 0), (12345, 3, 2), ((1 << 64) - 1, 2, 1), ((1 << 64) + 5, 2, 1),
        (2 ** 40 + 17, 1 << 20, (1 << 20) - 1),
    ]
    for seed, size, idx in cases:
        ss = R.RngStreamSet(size, seed)
        st = ss.stream(idx)
        ops = []
        for j in range(6):
            ops.append(["u01", None, st.uniform01().hex(), int(ss.counters[idx])])
        for j in range(6):
            ops.append(["normal", None, float(st.normal()).hex(), int(ss.counters[idx])])
        for shape in (0.3, 0.5, 1.0, 2.0, 10.0):
            for j in range(4):
                ops.append(["gamma", shape, float(st.gamma(shape)).hex(), int(ss.counters[idx])])
        g["streams"].append({"seed": str(seed), "size": size, "index": idx, "ops": ops})

    # fill_* batch variants (rng.py:120-135) -- the resampling-stream pattern.
    for seed, kind, n, shape in [(1306, "u01", 257, None), (7, "normal", 129, None),
                                 (99, "gamma", 65, 2.0), (99, "gamma", 65, 0.7)]:
        ss = R.RngStreamSet(4, seed)
        st = ss.stream(3)
        if kind == "u01":
            v = st.uniform01(n)
        elif kind == "normal":
            v = st.normal(0.0, 1.0, n)
        else:
            v = st.gamma(shape, 1.0, n)
        g["fills"].append({"seed": seed, "kind": kind, "n": n, "shape": shape, "stream": 3,
                           "values": hx(v), "counter": int(ss.counters[3])})

    # One draw from each of many streams (the per-particle kernel pattern).
    for seed, size, kind in [(1306, 4097, "u01"), (1306, 4097, "normal"), (5, 2049, "gamma2"),
                             (5, 2049, "gamma05")]:
        ss = R.RngStreamSet(size, seed)
        ctrs, k0, k1 = ss.counters, *ss.key
        vals = []
        for i in range(size):
            if kind == "u01":
                vals.append(R.u01(ctrs, i, k0, k1))
            elif kind == "normal":
                vals.append(R.std_normal(ctrs, i, k0, k1))
            elif kind == "gamma2":
                vals.append(R.std_gamma(ctrs, i, k0, k1, 2.0))
            else:
                vals.append(R.std_gamma(ctrs, i, k0, k1, 0.5))
        g["draw_sets"].append({"seed": seed, "size": size, "kind": kind, "values": hx(vals),
                               "counters": [int(c) for c in ctrs]})

    with open(out_path, "w") as f:
        json.dump(g, f, indent=None, separators=(",", ":"))
    print("wrote", out_path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "rng_golden.json"))
