"""The multi-rank bench path (torchrun, world size 2) end to end on ONE GPU: both ranks on
cuda:0 with host-staged gloo collectives (SMC_BENCH_FUNCTIONAL=1).  Checks that the sharded
filter runs through bench.py and reports a whole-job line; timings are not asserted."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_functional():
    env = dict(os.environ, SMC_BENCH_FUNCTIONAL="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--particles", "65536", "--no-cpu-baseline", "--no-e2e", "--no-gmm"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["n_particles"] == 2 * 65536
    assert line["value"] > 0 and line["resampled_frac"] == 1.0


@pytest.mark.parametrize("p2p", [1, 0])
def test_two_process_sharded_pf_bit_identical(p2p):
    """Two processes on cuda:0 (gloo for the small collectives): with p2p the cross-shard rows
    are read from the other process's memory through CUDA-IPC mappings (no host plan, no
    send / receive); the state must equal the single-GPU filter bit for bit."""
    env = dict(os.environ, SMC_DIST_GLOO="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29541 + p2p), os.path.join(ROOT, "tools", "dist_check.py"),
           "--p2p", str(p2p)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["ok"] and line["p2p"] == bool(p2p), line
