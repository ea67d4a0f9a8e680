"""world_size-2 gloo test of the replica aggregation used by bench.py (CPU)."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_00768_b200.replicas import aggregate

    secs, work = aggregate(1.5 + rank, 100.0 * (rank + 1))
    q.put((rank, secs, work))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    for _, secs, work in res:
        assert secs == 2.5 and work == 300.0


def test_single_process_is_identity():
    from paper_2309_00768_b200.replicas import aggregate

    assert aggregate(2.0, 7.0) == (2.0, 7.0)
