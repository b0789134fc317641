"""Id-sharded S-Merge / J-Merge across GPUs.

Partitioning: local rows (the ascending union of member ids) are split into
P contiguous ranges; rank r owns rows [lo_r, hi_r).  Vectors are replicated;
the k-NN lists are replicated between rounds.  One round:

1. every rank: reverse edges into its own rows, the hoods of its own
   vertices, and the local join over them (``knnm_round_local``), which
   leaves reference-order update slots for EVERY target row;
2. all-to-all (the only data-path exchange): rank s sends rank q the slot
   counts of q's rows and the contiguous slot range holding them;
3. every rank applies its rows from the P received blocks in source-rank
   order (``knnm_round_apply``).  Hood ids ascend with the rank, so
   source order is hood order, which is the reference's sequential order:
   the sharded result is bit-identical to the single-GPU one;
4. all-gather of the owned row blocks (lists replicated again) and
   all-reduce of the pair / accepted counters (convergence test, report).

The collectives run through a small communicator interface:
``TorchComm`` (torch.distributed: NCCL between GPUs, gloo on CPU) or
``LoopbackComm`` (P virtual ranks in one process -- used to run the full
sharded protocol on a single GPU in tests).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check
from .construct import MODE_CROSS, MODE_CROSS_OR_S2, BuildReport, RoundStats
from .core import DistanceCounter, Metric, sample_distinct
from .engine import Engine
from .graph import KnnGraph
from .merge import MergeParams, _check_merge_inputs, _merge_members, _sample_pool_rows


def shard_bounds(n: int, world: int):
    """Contiguous owned ranges [lo_r, hi_r) of the n local rows."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


# ---------------------------------------------------------------------------
# device views
# ---------------------------------------------------------------------------

class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can view engine memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None,
        }


def _view(ptr, shape, typestr, device):
    import torch

    if int(np.prod(shape)) == 0:
        dt = {"<f8": torch.float64, "<i4": torch.int32, "<i8": torch.int64, "|u1": torch.uint8}[typestr]
        return torch.empty(shape, dtype=dt, device=device)
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


class ShardEngine:
    """An Engine plus the sharded-round entry points of the C-ABI."""

    def __init__(self, engine: Engine):
        self.e = engine
        self.lib = engine._lib
        self.device = f"cuda:{engine.device}"

    def set_shard(self, lo, hi):
        check(self.lib.knnm_set_shard(self.e._h, int(lo), int(hi)), "knnm_set_shard")

    def round_local(self, mode, rev_cap, seed) -> int:
        p = ctypes.c_int64()
        check(self.lib.knnm_round_local(self.e._h, int(mode), int(rev_cap), ctypes.c_uint64(seed),
                                        ctypes.byref(p)), "knnm_round_local")
        return int(p.value)

    def local_views(self, n):
        """(cnt u32 (n,), boff u64 (n+1,), Bd f64, Bs i32) as torch views."""
        cnt, boff, bd, bs = (ctypes.c_void_p() for _ in range(4))
        check(self.lib.knnm_local_views(self.e._h, ctypes.byref(cnt), ctypes.byref(boff),
                                        ctypes.byref(bd), ctypes.byref(bs)), "knnm_local_views")
        boff_t = _view(boff.value, (n + 1,), "<i8", self.device)
        total = int(boff_t[n].item())
        # Bs is None when the slots are packed (source row inside Bd)
        return (_view(cnt.value, (n,), "<i4", self.device), boff_t,
                _view(bd.value, (max(total, 0),), "<f8", self.device),
                None if bs.value is None else _view(bs.value, (max(total, 0),), "<i4", self.device))

    def local_compact(self, n):
        """local_views over the written slots only (knnm_local_compact)."""
        cnt, boff, bd, bs = (ctypes.c_void_p() for _ in range(4))
        tot = ctypes.c_int64()
        check(self.lib.knnm_local_compact(self.e._h, ctypes.byref(cnt), ctypes.byref(boff),
                                          ctypes.byref(bd), ctypes.byref(bs), ctypes.byref(tot)),
              "knnm_local_compact")
        total = int(tot.value)
        return (_view(cnt.value, (n,), "<i4", self.device), _view(boff.value, (n + 1,), "<i8", self.device),
                _view(bd.value, (total,), "<f8", self.device),
                None if bs.value is None else _view(bs.value, (total,), "<i4", self.device))

    def round_apply(self, recv_cnt, recv_base, recv_bd, recv_bs) -> int:
        acc = ctypes.c_int64()
        base = np.ascontiguousarray(recv_base, dtype=np.uint64)
        check(self.lib.knnm_round_apply(
            self.e._h, len(base), ctypes.c_void_p(recv_cnt.data_ptr()),
            base.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(recv_bd.data_ptr()),
            ctypes.c_void_p(recv_bs.data_ptr()), ctypes.byref(acc)), "knnm_round_apply")
        return int(acc.value)

    def state_views(self, n, k):
        ids, dists, flags, sizes = (ctypes.c_void_p() for _ in range(4))
        check(self.lib.knnm_state_views(self.e._h, ctypes.byref(ids), ctypes.byref(dists),
                                        ctypes.byref(flags), ctypes.byref(sizes)), "knnm_state_views")
        return (_view(ids.value, (n, k), "<i4", self.device),
                _view(dists.value, (n, k), "<f8", self.device),
                _view(flags.value, (n, k), "|u1", self.device),
                _view(sizes.value, (n,), "<i4", self.device))

    def sync(self):
        self.e.sync()


# ---------------------------------------------------------------------------
# communicators: every call takes/returns {local_rank: value}
# ---------------------------------------------------------------------------

class LoopbackComm:
    """P virtual ranks in one process (all local)."""

    def __init__(self, world: int):
        self.world = int(world)
        self.local_ranks = list(range(self.world))

    def alltoallv(self, sends):
        """sends[s] = list of P tensors (to rank q); returns recv[q] = list of P (from s)."""
        return {q: [sends[s][q] for s in range(self.world)] for q in self.local_ranks}

    def allgather_blocks(self, fulls, bounds):
        """fulls[r] = list of full-size tensors; rank r's rows [lo_r, hi_r) are
        authoritative.  Afterwards every rank holds every block."""
        for q in self.local_ranks:
            for r in range(self.world):
                if r == q:
                    continue
                lo, hi = bounds[r]
                for tq, tr in zip(fulls[q], fulls[r]):
                    tq[lo:hi].copy_(tr[lo:hi])

    def allreduce_sum(self, vals):
        return int(sum(vals[r] for r in self.local_ranks))

    def barrier(self):
        pass


class TorchComm:
    """torch.distributed communicator (one rank per process; NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_ranks = [self.rank]

    def alltoallv(self, sends):
        import torch

        mine = sends[self.rank]
        dev = mine[0].device
        in_sizes = [int(t.numel()) for t in mine]
        sz = torch.tensor(in_sizes, dtype=torch.int64, device=dev)
        out_sz = torch.empty_like(sz)
        self.dist.all_to_all_single(out_sz, sz, group=self.group)
        out_sizes = [int(v) for v in out_sz.tolist()]
        inp = torch.cat([t.reshape(-1) for t in mine]) if sum(in_sizes) else torch.empty(0, dtype=mine[0].dtype, device=dev)
        out = torch.empty(sum(out_sizes), dtype=mine[0].dtype, device=dev)
        self.dist.all_to_all_single(out, inp, output_split_sizes=out_sizes,
                                    input_split_sizes=in_sizes, group=self.group)
        return {self.rank: list(torch.split(out, out_sizes))}

    def allgather_blocks(self, fulls, bounds):
        # row blocks of a C-contiguous (n, ...) tensor are contiguous views:
        # each owner broadcasts its block in place
        for t in fulls[self.rank]:
            for r in range(self.world):
                lo, hi = bounds[r]
                if hi > lo:
                    self.dist.broadcast(t[lo:hi], src=r, group=self.group)

    def allreduce_sum(self, vals):
        import torch

        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(vals[self.rank])], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# sharded round loop (construct.py:111-179)
# ---------------------------------------------------------------------------

def sharded_rounds(shards, comm, n, k, mode, params, rng, counter, report, rev_cap=None,
                   compact=True, traffic=None):
    """_descent_rounds over P ranks.  ``shards[r]`` = ShardEngine of each
    local rank r (state already initialised and replicated).  ``compact``:
    exchange only the written slots (unwritten ones can never be accepted);
    ``traffic`` (dict) accumulates the slot bytes each rank sends to others."""
    import torch

    from .construct import sample_cap

    cap = sample_cap(getattr(params, "rho", 1.0), k)
    rev_cap = cap if rev_cap is None else int(rev_cap)
    bounds = shard_bounds(n, comm.world)
    threshold = params.min_update_fraction * n * k
    for r in comm.local_ranks:
        shards[r].set_shard(*bounds[r])
        shards[r].e.set_sample(cap if cap < k else 0)
    for it in range(1, params.max_iters + 1):
        round_seed = int(rng.integers(0, 2**63 - 1))
        pairs_l = {r: shards[r].round_local(mode, rev_cap, round_seed) for r in comm.local_ranks}
        sends = {}
        for r in comm.local_ranks:
            cnt, boff, bd, bs = shards[r].local_compact(n) if compact else shards[r].local_views(n)
            boff_h = boff.cpu().numpy()
            parts = []
            for q, (lo, hi) in enumerate(bounds):
                a, b = int(boff_h[lo]), int(boff_h[hi])
                parts.append((cnt[lo:hi], bd[a:b], None if bs is None else bs[a:b]))
                if traffic is not None and q != r:
                    traffic[r] = traffic.get(r, 0) + (b - a) * (8 if bs is None else 12)
            sends[r] = parts
        recv_cnt = comm.alltoallv({r: [p[0] for p in sends[r]] for r in comm.local_ranks})
        recv_bd = comm.alltoallv({r: [p[1] for p in sends[r]] for r in comm.local_ranks})
        # packed slots (certified routes) carry the source row inside Bd
        packed = all(sends[r][0][2] is None for r in comm.local_ranks)
        recv_bs = None if packed else \
            comm.alltoallv({r: [p[2] for p in sends[r]] for r in comm.local_ranks})
        acc_l = {}
        for q in comm.local_ranks:
            sizes = [int(t.numel()) for t in recv_bd[q]]
            base = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype(np.uint64)
            rc = torch.cat([t.reshape(-1) for t in recv_cnt[q]]).contiguous()
            rb = torch.cat([t.reshape(-1) for t in recv_bd[q]]).contiguous() if sum(sizes) else \
                torch.empty(1, dtype=torch.float64, device=shards[q].device)
            rs = torch.cat([t.reshape(-1) for t in recv_bs[q]]).contiguous() \
                if (recv_bs is not None and sum(sizes)) else \
                torch.empty(1, dtype=torch.int32, device=shards[q].device)
            acc_l[q] = shards[q].round_apply(rc, base, rb, rs)
        fulls = {r: list(shards[r].state_views(n, k)) for r in comm.local_ranks}
        for r in comm.local_ranks:
            shards[r].sync()
        comm.allgather_blocks(fulls, bounds)
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        pairs = comm.allreduce_sum(pairs_l)
        accepted = comm.allreduce_sum(acc_l)
        if pairs > 0:
            counter.add(pairs)
        cur_phi = shards[comm.local_ranks[0]].e.phi()
        if report is not None:
            report.rounds.append(RoundStats(it, pairs, accepted, cur_phi, counter.count))
        if accepted <= threshold:
            if report is not None:
                report.converged = True
            return
    if report is not None:
        report.converged = False


# ---------------------------------------------------------------------------
# sharded merges: replicated initialisation, sharded rounds
# ---------------------------------------------------------------------------

def _append_random_all(engines, rows, pool, count, rng, counter):
    """merge.py:166-176 with identical draws applied to every local engine."""
    if count <= 0 or rows.size == 0 or pool.size == 0:
        return
    m, t = pool.shape[0], int(count)
    if t == m or 4 * t * t >= m:
        picks = _sample_pool_rows(rng, rows.size, count, pool).ravel().astype(np.int32)
        for e in engines:
            e.insert_rows(rows.astype(np.int32), count, picks)
    else:
        # every local engine replays the same PCG64 stream on the device
        st0 = rng.bit_generator.state
        for i, e in enumerate(engines):
            if i:
                rng.bit_generator.state = st0
            bad = e.draws_gen(rng, m, rows.size, t)
            while bad.size:
                bad = e.draws_regen(rng, m, bad)
            e.draws_insert(rows.astype(np.int32), pool.astype(np.int32))
    counter.add(rows.size * t)


def s_merge_sharded(dataset, g, h, params: MergeParams, comm, engines, counter=None,
                    return_report=False, out_device=False, compact=True, traffic=None):
    """s_merge (merge.py:195-260) over comm.world ranks; ``engines`` maps each
    local rank to an Engine.  Bit-identical to s_merge."""
    _check_merge_inputs(dataset, g, h.member_ids, params, h)
    counter = DistanceCounter() if counter is None else counter
    rng = np.random.default_rng(params.seed)
    metric = Metric(g.metric)
    k, k1 = params.k, params.k1
    union, rows_g, rows_h = _merge_members(np.asarray(g.member_ids), np.asarray(h.member_ids))
    n = union.shape[0]
    labels = np.zeros(n, dtype=np.int8)
    labels[rows_h] = 1
    local = [engines[r] for r in comm.local_ranks]
    for e in local:
        e.set_dataset(dataset.vectors, int(metric))
        e.begin(union, labels, k)
        e.load_graph(rows_g, g, k1)
        e.load_graph(rows_h, h, k1)
    fill = k - k1
    _append_random_all(local, rows_g, rows_h.astype(np.int64), min(fill, rows_h.size), rng, counter)
    _append_random_all(local, rows_h, rows_g.astype(np.int64), min(fill, rows_g.size), rng, counter)
    report = BuildReport(phi_initial=local[0].phi())
    shards = {r: ShardEngine(engines[r]) for r in comm.local_ranks}
    sharded_rounds(shards, comm, n, k, MODE_CROSS, params.descent_params(), rng, counter, report,
                   compact=compact, traffic=traffic)
    ids, dists, sizes = local[0].export(merge_rear=k - k1 > 0, on_device=out_device)
    u = KnnGraph.from_arrays(union, k, metric, ids, dists, sizes)
    return (u, report) if return_report else u


def j_merge_sharded(dataset, g, raw_ids, params: MergeParams, comm, engines, counter=None,
                    return_report=False, out_device=False, compact=True, traffic=None):
    """j_merge (merge.py:263-338) over comm.world ranks (non-empty raw set)."""
    raw = np.unique(np.asarray(raw_ids, dtype=np.int64))
    _check_merge_inputs(dataset, g, raw, params, None)
    if raw.size == 0:
        raise ValueError("use j_merge for an empty raw set")
    counter = DistanceCounter() if counter is None else counter
    rng = np.random.default_rng(params.seed)
    metric = Metric(g.metric)
    k, k1 = params.k, params.k1
    union, rows_g, rows_raw = _merge_members(np.asarray(g.member_ids), raw)
    n = union.shape[0]
    if k >= n:
        raise ValueError(f"k={k} must be below the union size {n}")
    labels = np.zeros(n, dtype=np.int8)
    labels[rows_raw] = 1
    local = [engines[r] for r in comm.local_ranks]
    for e in local:
        e.set_dataset(dataset.vectors, int(metric))
        e.begin(union, labels, k)
        e.load_graph(rows_g, g, k1)
    _append_random_all(local, rows_g, rows_raw.astype(np.int64), min(k - k1, rows_raw.size), rng,
                       counter)
    from .core import sample_distinct_rows

    init = sample_distinct_rows(rng, n, k, rows_raw)
    for e in local:
        e.insert_rows(rows_raw.astype(np.int32), k, init.ravel().astype(np.int32))
    counter.add(rows_raw.size * k)
    report = BuildReport(phi_initial=local[0].phi())
    shards = {r: ShardEngine(engines[r]) for r in comm.local_ranks}
    sharded_rounds(shards, comm, n, k, MODE_CROSS_OR_S2, params.descent_params(), rng, counter,
                   report, compact=compact, traffic=traffic)
    ids, dists, sizes = local[0].export(merge_rear=k - k1 > 0, on_device=out_device)
    u = KnnGraph.from_arrays(union, k, metric, ids, dists, sizes)
    return (u, report) if return_report else u
