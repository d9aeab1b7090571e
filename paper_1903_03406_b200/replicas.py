"""Multi-GPU: independent PLCs per GPU (BASELINE north_star: "refinement
itself does not shard").  One process per GPU; PLC k goes to rank
k % world; no collective touches the mesh -- ranks only exchange their
totals (Steiner points, device seconds) at the end (max-over-ranks time).
"""

from __future__ import annotations

import os
import queue
import threading
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


def refine_batch(plcs, cfg, device: int = None, streams: int = 4, prepared=None):
    """Refine independent PLCs on one GPU, ``streams`` at a time: each host
    thread drives its own context (own CUDA stream, caching allocator and
    counters), so the rounds of several PLCs overlap on the device -- one PLC
    of C5 keeps only a few SMs busy per round.  Returns the per-PLC
    (Mesh, QualityReport) pairs in input order (or GqCounts with
    ``prepared=(preps, keeps)``: the device-resident path)."""
    from concurrent.futures import ThreadPoolExecutor

    from . import _native
    from .refine import default_device, refine

    dev = default_device() if device is None else device
    streams = max(1, min(streams, len(plcs) if prepared is None else len(prepared[0])))
    pool = _contexts(dev, streams)
    free = queue.Queue()
    for c in pool:
        free.put(c)

    def one(i):
        ctx = free.get()
        try:
            if prepared is not None:
                prep, keep = prepared[0][i], prepared[1][i]
                return ctx.refine(prep, keep, cfg.B, cfg.max_rounds, cfg.seed)
            return refine(plcs[i], cfg, context=ctx)
        finally:
            free.put(ctx)

    n = len(plcs) if prepared is None else len(prepared[0])
    with ThreadPoolExecutor(max_workers=streams) as ex:
        return list(ex.map(one, range(n)))


_POOLS = {}
_POOL_LOCK = threading.Lock()


def _contexts(device: int, k: int):
    from . import _native
    with _POOL_LOCK:
        pool = _POOLS.setdefault(device, [])
        while len(pool) < k:
            pool.append(_native.Context(device))
        return pool[:k]
