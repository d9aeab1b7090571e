"""Multi-process (gloo, world_size 2) test of the replicas-only multi-GPU
driver: PLCs are split round-robin, totals combined with max-over-ranks time."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_1903_03406_b200 import synth
    from paper_1903_03406_b200.replicas import my_share, run_replicas

    plcs = [synth.cube_points(5 + k, k) for k in range(5)]

    def cpu_worker(plc, B):
        o = oracle.refine(plc, B=B)
        return int((o["vert_origin"] == 1).sum()), 0.01 * (1 + rank)

    res = run_replicas(plcs, 2.0, worker=cpu_worker)
    out[rank] = (res["steiner"], res["seconds"], res["plcs"], my_share(5, rank, world))
    dist.destroy_process_group()


def test_replicas_two_ranks_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle
    from paper_1903_03406_b200 import synth
    total = sum(int((oracle.refine(synth.cube_points(5 + k, k), B=2.0)["vert_origin"] == 1).sum()) for k in range(5))
    assert out[0][0] == out[1][0] == total          # every rank sees the job total
    assert out[0][2] == out[1][2] == 5
    assert abs(out[0][1] - 0.02 * 2) < 1e-12         # max over ranks of per-rank time (rank 1: 2 PLCs x 0.02)
    assert out[0][3] == [0, 2, 4] and out[1][3] == [1, 3]


def _gpu_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), GQM3D_DEVICE="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1903_03406_b200 import synth
    from paper_1903_03406_b200.replicas import run_replicas
    plcs = [synth.cube_points(300 + 50 * k, k) for k in range(4)]
    res = run_replicas(plcs, 1.5)          # default worker: the GPU refine()
    out[rank] = (res["steiner"], res["plcs"])
    dist.destroy_process_group()


@pytest.mark.gpu
def test_replicas_two_ranks_gpu_path():
    """The multi-process driver with the real GPU worker: two ranks (gloo for
    the totals, both on the one B200 of this box -- independent PLCs, no
    kernel of one rank waits on the other), totals equal the single-process sum."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from paper_1903_03406_b200 import RefineConfig, refine, synth
    total = sum(refine(synth.cube_points(300 + 50 * k, k), RefineConfig(B=1.5))[1].steiner_points for k in range(4))
    assert out[0][0] == out[1][0] == total
    assert out[0][1] == out[1][1] == 4
