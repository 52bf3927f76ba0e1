"""Multi-rank host logic on CPU (world size 2, gloo): the collectives the sharded
sampler uses, the exchange plan every rank derives from allgathered counts, and
the rank-order combine of normalization partials.  The device kernels of the
sharded path are checked on one GPU in tests/test_gpu_dist.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1306_5583_b200.dist import TorchComm, combine_partials_reference, exchange_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        rng = np.random.default_rng(7)  # same global counts on every rank
        n = 1000
        counts = rng.multinomial(n * world, np.full(n * world, 1.0 / (n * world))).astype(np.int64)
        mine = counts[rank * n:(rank + 1) * n]
        z = int((mine == 0).sum())
        s = int(np.maximum(mine - 1, 0).sum())
        zsp = comm.allgather(torch.tensor([z, s, int((mine >= 2).sum()), 1], dtype=torch.int32))
        zsp = zsp.numpy()
        plans = exchange_plan(zsp[:, 0], zsp[:, 1])
        plan = plans[rank]
        # send the global surplus ranks (as payload) and check the receiver gets what the pairing says
        sends = [(p, torch.arange(plan["soff"] + lo, plan["soff"] + lo + c, dtype=torch.float64).reshape(-1, 1))
                 for p, lo, c in plan["sends"]]
        recvs = [(p, torch.empty((c, 1), dtype=torch.float64)) for p, c in plan["recvs"]]
        comm.exchange(sends, recvs)
        got = torch.cat([t for _, t in recvs]).ravel().numpy() if recvs else np.zeros(0)
        # expected: my zero ranks outside my own surplus range, ascending
        my_ranks = np.arange(plan["zoff"], plan["zoff"] + z)
        remote = my_ranks[(my_ranks < plan["soff"]) | (my_ranks >= plan["soff"] + plan["s_self"])]
        ok_exchange = np.array_equal(got, remote)
        # normalization partials: rank-order combine equals the single-system normalization
        lw = np.random.default_rng(11).normal(0, 3, n * world)
        part = lw[rank * n:(rank + 1) * n]
        m = part.max()
        e = np.exp(part - m)
        p8 = torch.tensor([m, e.sum(), (e * e).sum(), 0, 0, 0, 0, 0], dtype=torch.float64)
        allp = comm.allgather(p8).numpy()
        c = combine_partials_reference(allp)
        M = lw.max()
        E = np.exp(lw - M)
        ok_combine = abs(c["lse"] - (M + np.log(E.sum()))) < 1e-12 and abs(c["ess"] - E.sum() ** 2 / (E * E).sum()) \
            < 1e-9 * c["ess"]
        q.put((rank, ok_exchange, ok_combine, len(plan["sends"]), len(plan["recvs"])))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_and_combine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res


@pytest.mark.parametrize("G", [2, 3, 8])
def test_exchange_plan_properties(G):
    rng = np.random.default_rng(G)
    n = 257
    counts = rng.multinomial(n * G, rng.dirichlet(np.full(n * G, 0.3))).astype(np.int64)
    Z = [int((counts[g * n:(g + 1) * n] == 0).sum()) for g in range(G)]
    S = [int(np.maximum(counts[g * n:(g + 1) * n] - 1, 0).sum()) for g in range(G)]
    plans = exchange_plan(Z, S)
    for g in range(G):
        for h, lo, c in plans[g]["sends"]:
            assert (g, c) in [(p, k) for p, k in plans[h]["recvs"]]
        local = max(0, min(plans[g]["zoff"] + Z[g], plans[g]["soff"] + S[g]) - max(plans[g]["zoff"], plans[g]["soff"]))
        assert local + sum(c for _, c in plans[g]["recvs"]) == Z[g]
    with pytest.raises(ValueError):
        exchange_plan([1, 0], [0, 0])
