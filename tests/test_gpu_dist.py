"""Sharded (multi-GPU) resampling kernels, emulated as G logical shards on ONE GPU:
per-shard counts, the global parent pairing and the cross-shard row exchange
must reproduce the single-system result bit for bit."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SCHEMES = ["multinomial", "residual", "stratified", "systematic", "residual_stratified", "residual_systematic"]


def _ws(n):
    from paper_1306_5583_b200 import _abi
    return torch.empty(_abi.lib().smc_resample_workspace_bytes(n), dtype=torch.uint8, device="cuda")


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("G,n,kind", [(2, 3000, "heavy"), (4, 2048, "heavy"), (3, 5001, "heavy"), (8, 700, "heavy"),
                                      (4, 4096, "last_shard"), (3, 2500, "first_shard")])
def test_sharded_resample_equals_single(scheme, G, n, kind):
    from paper_1306_5583_b200 import _abi
    from paper_1306_5583_b200.dist import exchange_plan
    from paper_1306_5583_b200.resample import _scheme

    sid = int(_scheme(scheme))
    N = G * n
    rng = np.random.default_rng(N + sid)
    lw = rng.normal(0, 2.5, N)
    if kind == "heavy":
        lw[rng.integers(N)] += 6.0  # one heavy particle: lots of cross-shard surplus
    elif kind == "last_shard":  # (almost) all weight on the last shard: its surplus ranks run far past n
        lw[:-n] -= 40.0
    else:  # ... or on the first: every other shard is all zero slots
        lw[n:] -= 40.0
    w = O.normalize_log(lw)[1]
    u = rng.random(N)
    x = rng.normal(size=(N, 4))
    counts_ref, _ = O.resample_counts(scheme, w, u=u)
    x_ref = O.copy_rows(x.copy(), O.replication_to_parents(counts_ref))

    ug = torch.as_tensor(u).cuda()
    st = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(G)]
    ws = [_ws(n) for _ in range(G)]
    wg = [torch.as_tensor(w[g * n:(g + 1) * n]).cuda().contiguous() for g in range(G)]
    xg = [torch.as_tensor(x[g * n:(g + 1) * n]).cuda().contiguous() for g in range(G)]
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    S = _abi.stream()
    totals = []
    for g in range(G):
        t = torch.zeros(4, dtype=torch.int64, device="cuda")
        _abi.call("smc_resample_shard_totals", sid, p(wg[g]), None, None, n, N, N, p(ug), N, None, p(st[g]), p(ws[g]),
                  ws[g].numel(), p(t), S)
        totals.append(t)
    totals_all = torch.cat(totals)
    counts, zsp = [], []
    for g in range(G):
        c = torch.empty(n, dtype=torch.int32, device="cuda")
        z = torch.zeros(4, dtype=torch.int32, device="cuda")
        _abi.call("smc_resample_shard_counts", sid, p(wg[g]), None, None, n, N, N, G, g, p(totals_all), 0, N, None,
                  p(ug), N, p(c), None, p(st[g]), p(ws[g]), ws[g].numel(), p(z), S)
        counts.append(c)
        zsp.append(z)
    assert all(int(s.item()) == 0 for s in st)
    got = torch.cat(counts).cpu().numpy()
    assert np.array_equal(got, counts_ref)  # bit-identical to one GPU
    zsp = torch.stack(zsp).cpu().numpy()
    plans = exchange_plan(zsp[:, 0], zsp[:, 1])
    # pack on every sender, route slices to receivers in peer order
    outbox = {}
    for g in range(G):
        sends = plans[g]["sends"]
        tot = sum(c for _, _, c in sends)
        buf = torch.empty((max(tot, 1), 4), dtype=torch.float64, device="cuda")
        if tot:
            ranges = (ctypes.c_int64 * (2 * len(sends)))(*[v for _, lo, c in sends for v in (lo, c)])
            _abi.call("smc_resample_shard_pack", p(xg[g]), 32, n, ranges, len(sends), p(buf), p(ws[g]), ws[g].numel(),
                      S)
        o = 0
        for peer, _, c in sends:
            outbox[(g, peer)] = buf[o:o + c]
            o += c
    new = []
    for g in range(G):
        parts = [outbox[(h, g)] for h, _ in plans[g]["recvs"]]
        recv = torch.cat(parts).contiguous() if parts else None
        par = torch.empty(n, dtype=torch.int32, device="cuda")
        _abi.call("smc_resample_shard_assign", p(counts[g]), n, plans[g]["zoff"], plans[g]["soff"], plans[g]["s_self"],
                  None if recv is None else p(recv), p(xg[g]), 32, p(par), p(ws[g]), ws[g].numel(), S)
        new.append(xg[g][par.long()])  # the gather the next move performs
    assert np.array_equal(torch.cat(new).cpu().numpy(), x_ref)
