"""World-size-2 gloo tests (CPU) of the torch.distributed communicator that
carries the sharded rounds between GPUs (paper_1908_00814_b200/distributed.py):
uneven all-to-all of slot blocks, in-place all-gather of owned row blocks,
all-reduce of counters, and the shard bounds."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1908_00814_b200.distributed import TorchComm, shard_bounds

        comm = TorchComm()
        # uneven all-to-all: rank s sends (s+1)*(q+1) elements valued 100*s+q to q
        sends = [torch.full(((rank + 1) * (d + 1),), 100 * rank + d, dtype=torch.float64)
                 for d in range(world)]
        sends[1 % world] = torch.empty(0, dtype=torch.float64) if rank == 0 else sends[1 % world]
        recv = comm.alltoallv({rank: sends})[rank]
        ok_a2a = True
        for s in range(world):
            exp = 0 if (s == 0 and rank == 1 % world) else (s + 1) * (rank + 1)
            ok_a2a &= recv[s].numel() == exp and bool(torch.all(recv[s] == 100 * s + rank))
        # all-gather of owned row blocks into replicated (n, k) arrays
        n, k = 11, 3
        bounds = shard_bounds(n, world)
        full = torch.full((n, k), -1, dtype=torch.int32)
        lo, hi = bounds[rank]
        full[lo:hi] = torch.arange(lo * k, hi * k, dtype=torch.int32).reshape(-1, k)
        comm.allgather_blocks({rank: [full]}, bounds)
        ok_ag = bool(torch.equal(full, torch.arange(n * k, dtype=torch.int32).reshape(n, k)))
        ok_ar = comm.allreduce_sum({rank: rank + 5}) == sum(r + 5 for r in range(world))
        q.put((rank, ok_a2a, ok_ag, ok_ar))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_torchcomm_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
    assert all(p.exitcode == 0 for p in procs)
    for rank, a2a, ag, ar in res:
        assert a2a and ag and ar, (rank, a2a, ag, ar)


def test_shard_bounds_cover_rows():
    from paper_1908_00814_b200.distributed import shard_bounds

    for n in (1, 7, 1000, 1000003):
        for world in (1, 2, 3, 8):
            b = shard_bounds(n, world)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert all(hi >= lo for lo, hi in b)
