"""Multi-GPU: independent PLCs per GPU (BASELINE north_star: "refinement
itself does not shard").  One process per GPU; PLC k goes to rank
k % world; no collective touches the mesh -- ranks only exchange their
totals (Steiner points, device seconds) at the end (max-over-ranks time).
"""

from __future__ import annotations

import os
import time


def my_share(n_items: int, rank: int, world: int):
    return list(range(rank, n_items, world))


def run_replicas(plcs, B: float, worker=None, group=None):
    """Refine every PLC assigned to this rank; returns the job totals
    {steiner, seconds (max over ranks), plcs} on every rank.  `worker(plc, B)`
    returns (steiner, seconds); default = the GPU refine()."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if worker is None:
        from .refine import refine
        from .config import RefineConfig

        def worker(plc, B):
            t = time.perf_counter()
            _, rep = refine(plc, RefineConfig(B=B))
            return rep.steiner_points, rep.device.get("device_ms", 1000 * (time.perf_counter() - t)) / 1000.0

    steiner, secs = 0, 0.0
    mine = my_share(len(plcs), rank, world)
    for k in mine:
        s, t = worker(plcs[k], B)
        steiner += int(s)
        secs += float(t)
    if world > 1:
        backend = dist.get_backend(group)
        if backend == "nccl":
            from .refine import default_device
            dev = torch.device("cuda", default_device())   # this rank's GPU (LOCAL_RANK)
            torch.cuda.set_device(dev)
        else:
            dev = torch.device("cpu")
        tt = torch.tensor([secs], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        ss = torch.tensor([steiner, len(mine)], dtype=torch.float64, device=dev)
        dist.all_reduce(ss, group=group)
        secs, steiner, n = float(tt[0]), int(ss[0]), int(ss[1])
    else:
        n = len(mine)
    return {"steiner": steiner, "seconds": secs, "plcs": n, "world": world}
