"""World-size-2 gloo tests (CPU) of the torch.distributed communicator that
carries the sharded rounds between GPUs (paper_1908_00814_b200/distributed.py):
the packed uneven exchange of slot blocks (with the chunk-count header), the
counter and row-record all-gathers, the in-place all-gather of owned row
blocks, all-reduce, the shard bounds and the tree's groups."""

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
        # uneven exchange of (count, slot, source) parts: rank s sends
        # (s+1)*(q+1) slots valued 100*s+q to q; rank 0 sends nothing to 1
        sends = []
        for dd in range(world):
            m = 0 if (rank == 0 and dd == 1 % world) else (rank + 1) * (dd + 1)
            sends.append([torch.full((3,), m, dtype=torch.int32),
                          torch.full((m,), 100 * rank + dd, dtype=torch.float64),
                          torch.arange(m, dtype=torch.int32)])
        recv, mx = comm.exchange({rank: sends}, {rank: 7 + rank})
        recv = recv[rank]
        ok_a2a = mx == 7 + world - 1
        for s in range(world):
            exp = 0 if (s == 0 and rank == 1 % world) else (s + 1) * (rank + 1)
            cnt, bd, bs = recv[s]
            ok_a2a &= bool(torch.all(cnt == exp)) and bd.numel() == exp and bs.numel() == exp
            ok_a2a &= bool(torch.all(bd == 100 * s + rank)) and bool(torch.equal(bs, torch.arange(exp, dtype=torch.int32)))
        # packed slots: a None part is skipped on both sides
        recv2, _ = comm.exchange({rank: [[t[0], t[1], None] for t in sends]}, {rank: 0})
        ok_a2a &= all(p[2] is None for p in recv2[rank])
        # counters and row records
        st = comm.allgather_counts({rank: [rank + 1, 10 * rank]})
        ok_ag = st.tolist() == [[r + 1, 10 * r] for r in range(world)]
        buf = torch.full(((rank + 1) * 16,), rank, dtype=torch.uint8)
        rows = comm.allgather_bytes({rank: buf}, st[:, 0], 16)[rank]
        ok_ag &= all(rows[s].numel() == (s + 1) * 16 and bool(torch.all(rows[s] == s))
                     for s in range(world))
        # all-gather of owned row blocks into replicated (n, k) arrays
        n, k = 11, 3
        bounds = shard_bounds(n, world)
        full = torch.full((n, k), -1, dtype=torch.int32)
        lo, hi = bounds[rank]
        full[lo:hi] = torch.arange(lo * k, hi * k, dtype=torch.int32).reshape(-1, k)
        comm.allgather_blocks({rank: [full]}, bounds)
        ok_ag &= bool(torch.equal(full, torch.arange(n * k, dtype=torch.int32).reshape(n, k)))
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


def test_tree_groups():
    from paper_1908_00814_b200.distributed import tree_groups

    g = tree_groups(8)
    assert [lv for lv, _ in g] == [1, 1, 1, 1, 2, 2, 3]
    assert g[-1][1] == list(range(8)) and g[0][1] == [0, 1] and g[5][1] == [4, 5, 6, 7]
    assert tree_groups(1) == []
    with pytest.raises(ValueError):
        tree_groups(6)
