"""Multi-process check of the sharded particle filter (torchrun; gloo on ONE GPU or NCCL on G).

Every rank runs its shard of a G-rank filter (the P2P exchange by default: cross-shard rows read
from the peers' memory through CUDA-IPC mappings); rank 0 also runs the unsharded filter of G*n
particles and compares: identical resampling decisions and a bit-identical state.

    SMC_DIST_GLOO=1 python -m torch.distributed.run --nproc-per-node 2 tools/dist_check.py [--p2p 0|1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 15)
    ap.add_argument("--steps", type=int, default=25)
    ap.add_argument("--scheme", default="systematic")
    ap.add_argument("--p2p", type=int, default=1)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    gloo = os.environ.get("SMC_DIST_GLOO") == "1"
    local = 0 if gloo else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1306_5583_b200 import pf
    from paper_1306_5583_b200.dist import Shard, TorchComm
    obs, _ = pf.generate_observations(args.steps + 1, 1306)
    shard = Shard(args.n, TorchComm())
    shard.p2p = None if args.p2p else False
    s = pf.make_sampler(args.n, args.scheme, 0.5, seed=1306, shard=shard)
    s.initialize(obs)
    s.iterate(args.steps)
    h = s.history()
    x = s.system.value.data.cpu()
    parts = [torch.empty_like(x) for _ in range(world)] if gloo else None
    if gloo:
        dist.all_gather(parts, x)
    else:
        xs = x.cuda()
        out = torch.empty((world,) + tuple(xs.shape), dtype=xs.dtype, device="cuda")
        dist.all_gather_into_tensor(out, xs)
        parts = list(out.cpu().unbind(0))
    if rank == 0:
        ref = pf.make_sampler(world * args.n, args.scheme, 0.5, seed=1306)
        ref.initialize(obs)
        ref.iterate(args.steps)
        href = ref.history()
        xref = ref.system.value.data.cpu().numpy()
        xs = torch.cat(parts).numpy()
        ok = bool(np.array_equal(h["resampled"], href["resampled"]) and np.array_equal(xs, xref)
                  and abs(s.log_zconst - ref.log_zconst) <= 1e-9 * abs(ref.log_zconst))
        print(json.dumps({"ok": ok, "p2p": bool(shard.p2p), "world": world, "n_per_rank": args.n,
                          "rows_differ": int((xs != xref).any(1).sum())}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
