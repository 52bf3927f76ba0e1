"""Particle sharding over GPUs (the role of vSMC's MPI module,
PAPER.md:1990-2059, on NCCL over NVLink).

Rank g of G holds particles [g n, (g+1) n) of N = G n.  Stream indices stay
global (the Philox stream of local particle i is g n + i) and the resampling
stream N is replicated on every rank, so every draw is the one a single GPU
would make.  Per step the ranks exchange only:

* the normalization partials {max, sum e, sum e^2, monitor} (8 doubles):
  allgathered and combined in RANK ORDER on every rank (bit-identical global
  weight state, unlike a reduction whose order depends on the algorithm);
* the resample totals {T lo, T hi, sum f, T'} (4 u64): exact integer offsets,
  so counts are bit-identical to one GPU;
* {zero slots, surplus children, surplus parents} (4 u32) -- from which every
  rank derives the same exchange plan -- and the rows of surplus children
  whose partner zero slot lives on another rank (grouped send/recv).

Survivors never move, so every rank keeps exactly n rows (load stays balanced).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi

__all__ = ["Shard", "TorchComm", "exchange_plan", "combine_partials_reference"]

PARTIAL_STRIDE = 8  # SMC_PARTIAL_STRIDE


def exchange_plan(Z, S):
    """Cross-shard pairing of zero slots and surplus children (SPEC.md:168 sweep, global ranks).

    Z[g], S[g]: zero slots / surplus children on rank g (sum Z == sum S).
    Returns per rank g: dict(zoff, soff, s_self, sends=[(peer, local_lo, count)],
    recvs=[(peer, count)]) -- sends/recvs ordered by peer, i.e. by global rank.
    """
    Z = [int(z) for z in Z]
    S = [int(s) for s in S]
    if sum(Z) != sum(S):
        raise ValueError("zero slots and surplus children do not pair up (counts do not sum to N)")
    G = len(Z)
    zoff = np.concatenate([[0], np.cumsum(Z)[:-1]]).astype(np.int64)
    soff = np.concatenate([[0], np.cumsum(S)[:-1]]).astype(np.int64)
    plans = []
    for g in range(G):
        sends, recvs = [], []
        for h in range(G):
            if h == g:
                continue
            # my zero ranks x rank h's surplus ranks -> rows h sends me
            a, b = max(zoff[g], soff[h]), min(zoff[g] + Z[g], soff[h] + S[h])
            if b > a:
                recvs.append((h, int(b - a)))
            # rank h's zero ranks x my surplus ranks -> rows I send to h
            a, b = max(zoff[h], soff[g]), min(zoff[h] + Z[h], soff[g] + S[g])
            if b > a:
                sends.append((h, int(a - soff[g]), int(b - a)))
        plans.append(dict(zoff=int(zoff[g]), soff=int(soff[g]), s_self=S[g], sends=sends, recvs=recvs))
    return plans


def combine_partials_reference(parts):
    """numpy statement of smc_weights_combine (rank-order two-phase combine), for tests."""
    parts = np.asarray(parts, dtype=np.float64).reshape(-1, PARTIAL_STRIDE)
    M = parts[:, 0].max()
    s1 = s2 = h0 = h1 = 0.0
    for p in parts:
        if p[0] != -np.inf:
            f = np.exp(p[0] - M)
            s1 += p[1] * f
            s2 += p[2] * (f * f)
        h0 += p[3]
        h1 += p[4]
    return dict(max=M, log_sum=np.log(s1), lse=M + np.log(s1), ess=s1 * s1 / s2, monitor=(h0, h1))


class TorchComm:
    """torch.distributed plumbing (NCCL on GPUs, gloo on CPU for the tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves host memory only: CUDA tensors are staged through the host (CPU tests and
        # the one-GPU functional check of the multi-rank bench); NCCL takes device memory
        self.staged = dist.get_backend(group) == "gloo"

    def allgather(self, t):
        if self.staged:
            h = t.detach().cpu().contiguous()
            out = torch.empty((self.world,) + tuple(h.shape), dtype=h.dtype)
            self.dist.all_gather(list(out.unbind(0)), h, group=self.group)
            return out.to(t.device)
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def peer_pointers(self, tensors):
        """Device addresses of every rank's `tensors` (same list on every rank), mapped into this
        process with CUDA IPC: rank r's entries are P2P-readable over NVLink (same-device
        processes work too).  Returns [rank][k] -> int address; the own rank's are its own."""
        mine = [(t.untyped_storage()._share_cuda_(), t.storage_offset() * t.element_size()) for t in tensors]
        allv = [None] * self.world
        self.dist.all_gather_object(allv, mine, group=self.group)
        self._ipc = getattr(self, "_ipc", [])
        out = []
        for r, entries in enumerate(allv):
            if r == self.rank:
                out.append([t.data_ptr() for t in tensors])
                continue
            row = []
            for handle, off in entries:
                st = torch.UntypedStorage._new_shared_cuda(*handle)
                self._ipc.append(st)  # keep the mapping alive
                row.append(st.data_ptr() + off)
            out.append(row)
        return out

    def exchange(self, sends, recvs):
        """sends: [(peer, tensor)], recvs: [(peer, tensor)] -- one grouped send/recv round."""
        if self.staged:
            hs = [(p, t.detach().cpu().contiguous()) for p, t in sends if t.numel()]
            hr = [(p, t, torch.empty(t.shape, dtype=t.dtype)) for p, t in recvs if t.numel()]
            ops = [self.dist.P2POp(self.dist.isend, h, p, group=self.group) for p, h in hs]
            ops += [self.dist.P2POp(self.dist.irecv, h, p, group=self.group) for p, _, h in hr]
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            for _, t, h in hr:
                t.copy_(h)
            return
        ops = [self.dist.P2POp(self.dist.isend, t, p, group=self.group) for p, t in sends if t.numel()]
        ops += [self.dist.P2POp(self.dist.irecv, t, p, group=self.group) for p, t in recvs if t.numel()]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()


class Shard:
    """This rank's slice of a G-rank particle system."""

    def __init__(self, n_local, comm):
        self.n = int(n_local)
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.n_total = self.n * self.world
        self.base = self.rank * self.n
        dev = torch.device("cuda", torch.cuda.current_device())
        self.partial = torch.zeros(PARTIAL_STRIDE, dtype=torch.float64, device=dev)
        self.totals = torch.zeros(4, dtype=torch.int64, device=dev)
        self.zsp = torch.zeros(4, dtype=torch.int32, device=dev)
        self.last_plan = None

    # -- normalization ------------------------------------------------------
    def combine(self, weight_set, mode, accumulate_nc, monitor_out=None):
        parts = self.comm.allgather(self.partial)
        _abi.call("smc_weights_combine", _abi.ptr(parts), self.world, weight_set.state_ptr, self.n_total, int(mode),
                  int(bool(accumulate_nc)), monitor_out, _abi.stream())

    # -- resampling ----------------------------------------------------------
    # p2p: cross-shard rows are read straight from the peers' memory by the assignment kernel
    # (CUDA IPC + NVLink loads; every offset from the allgathered counts on the device): no host
    # plan, no host synchronization and no send / receive per step.  None = decide on first use
    # (the communicator must offer peer_pointers); False = the host-planned send / receive path.
    p2p = None

    def _peer_table(self, system, buf):
        """IPC mappings of every rank's resample workspace and both state buffers (set up once;
        again only if a buffer moved)."""
        value = system.value
        value.alt()  # both halves of the double buffer exist before they are shared
        tensors = [system.resampler._ws.buf, value._bufs[0], value._bufs[1]]
        key = tuple(t.data_ptr() for t in tensors)
        if getattr(self, "_peer_key", None) != key:
            self._peers = self.comm.peer_pointers(tensors)
            self._peer_key = key
        return self._peers

    def resample(self, system, scheme, gate, status, rows, row_bytes):
        """Global resample of this shard's particles; returns True when it ran (host-planned
        path) or None (P2P path: whether it ran is decided on the device)."""
        ws_set = system.weight_set
        r = system.resampler
        n = self.n
        buf, nb = r._ws.get(_abi.lib().smc_resample_workspace_bytes(n))
        lw, st = _abi.ptr(ws_set.lw_raw), ws_set.state_ptr
        _abi.call("smc_resample_shard_totals", int(scheme), None, lw, st, n, self.n_total, self.n_total, None, 0,
                  gate, status, buf, nb, _abi.ptr(self.totals), _abi.stream())
        totals_all = self.comm.allgather(self.totals)
        ctr = system.rng_set.counter_ptr(n)  # the replicated resampling stream (global index N)
        _abi.call("smc_resample_shard_counts", int(scheme), None, lw, st, n, self.n_total, self.n_total, self.world,
                  self.rank, _abi.ptr(totals_all), system.rng_set.seed, self.n_total, ctr, None, 0, None, gate,
                  status, buf, nb, _abi.ptr(self.zsp), _abi.stream())
        zsp_dev = self.comm.allgather(self.zsp)  # (G, 4) {zero slots, surplus children, surplus parents, active}
        if self.p2p is None:
            self.p2p = hasattr(self.comm, "peer_pointers") and self.world <= 16
        if self.p2p:
            peers = self._peer_table(system, buf)
            cur = system.value._cur
            ws_arr = (ctypes.c_void_p * self.world)(*[peers[g][0] for g in range(self.world)])
            rows_arr = (ctypes.c_void_p * self.world)(*[peers[g][1 + cur] for g in range(self.world)])
            _abi.call("smc_resample_shard_assign_p2p", _abi.ptr(zsp_dev.contiguous()), self.world, self.rank, ws_arr,
                      rows_arr, n, rows, row_bytes, _abi.ptr(system.parents), status, buf, nb, _abi.stream())
            self.last_plan = None
            return None
        zsp_all = zsp_dev.cpu().numpy().reshape(self.world, 4)  # the host-planned path's one host sync
        if not zsp_all[self.rank, 3]:
            return False
        plan = exchange_plan(zsp_all[:, 0], zsp_all[:, 1])[self.rank]
        self.last_plan = plan
        dev = system.device
        sends = []
        nsend = sum(c for _, _, c in plan["sends"])
        if nsend:
            sendbuf = torch.empty((nsend, row_bytes // 8), dtype=torch.float64, device=dev)
            ranges = (ctypes.c_int64 * (2 * len(plan["sends"])))(
                *[v for _, lo, c in plan["sends"] for v in (lo, c)])
            _abi.call("smc_resample_shard_pack", rows, row_bytes, n, ranges, len(plan["sends"]), _abi.ptr(sendbuf),
                      buf, nb, _abi.stream())
            o = 0
            for peer, _, c in plan["sends"]:
                sends.append((peer, sendbuf[o:o + c]))
                o += c
        nrecv = sum(c for _, c in plan["recvs"])
        recvbuf = torch.empty((max(nrecv, 1), row_bytes // 8), dtype=torch.float64, device=dev)
        recvs, o = [], 0
        for peer, c in plan["recvs"]:
            recvs.append((peer, recvbuf[o:o + c]))
            o += c
        self.comm.exchange(sends, recvs)
        _abi.call("smc_resample_shard_assign", None, n, plan["zoff"], plan["soff"], plan["s_self"],
                  _abi.ptr(recvbuf) if nrecv else None, rows, row_bytes, _abi.ptr(system.parents), buf, nb,
                  _abi.stream())
        return True
