"""Id-sharded S-Merge / J-Merge across GPUs, and the multi-way tree merge
(SURVEY.md §8e).

Partitioning: local rows (the ascending union of member ids) are split into
P contiguous ranges; rank r owns rows [lo_r, hi_r).  Vectors are replicated;
the k-NN lists are replicated between rounds, the rear lists (merge_rear
tails) and the initialisation are sharded.

Initialisation (merge.py:217-256 / 297-325): every rank loads only the input
rows it owns and inserts only their random cross appends / raw-row draws
(the PCG64 draw matrices are generated for all rows, so the stream advances
exactly as the reference's), then the owned rows are all-gathered once.  A
rank therefore never needs the other ranks' input graphs: in the tree merge
each GPU keeps its own rows at every level and nothing is re-sharded.

One round (construct.py:111-179):

1. every rank: reverse edges into its own rows, the hoods of its own
   vertices (``knnm_round_local``), then the local join per hood chunk
   (``knnm_local_join``; one chunk unless the round's slots exceed the
   candidate budget), which leaves reference-order update slots for EVERY
   target row, compacted to the written ones (``knnm_local_compact``);
2. per chunk, one all-to-all of the slot blocks (rank s sends rank q the
   slot counts of q's rows and their slots, packed into one byte buffer; the
   size header also carries each rank's chunk count);
3. every rank applies its rows from the received blocks in (source rank,
   chunk) order (``knnm_round_apply``).  Hood ids ascend with the rank and
   with the chunk, so that is hood order, the reference's sequential order:
   the sharded result is bit-identical to the single-GPU one;
4. one all-gather of per-rank counters (pairs, accepted, changed rows) and
   one all-gather of the changed owned rows only (``knnm_pack_rows`` /
   ``knnm_unpack_rows``: rows whose flags the assembly cleared or that
   accepted an insert), so the next round starts from replicated lists.
   phi is reduced on each engine's side stream and read after the loop.

Collectives per round: 2 per hood chunk + 2.  Host reads per round in this
module: the slot split sizes per chunk and the counter all-gather.

The collectives run through a small communicator interface:
``TorchComm`` (torch.distributed: NCCL between GPUs; gloo with CPU staging
for tests) or ``LoopbackComm`` (P virtual ranks in one process -- used to
run the full sharded protocol on a single GPU in tests).
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace

import numpy as np

from ._lib import check
from .construct import MODE_CROSS, MODE_CROSS_OR_S2, BuildReport, RoundStats
from .core import DistanceCounter, Metric
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


_DT = {"<f8": "float64", "<i4": "int32", "<i8": "int64", "|u1": "uint8"}


def _view(ptr, shape, typestr, device):
    import torch

    if int(np.prod(shape)) == 0:
        return torch.empty(shape, dtype=getattr(torch, _DT[typestr]), device=device)
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


class ShardEngine:
    """An Engine plus the sharded-round entry points of the C-ABI."""

    def __init__(self, engine: Engine):
        self.e = engine
        self.lib = engine._lib
        self.device = f"cuda:{engine.device}"

    def set_shard(self, lo, hi):
        check(self.lib.knnm_set_shard(self.e._h, int(lo), int(hi)), "knnm_set_shard")
        self.lo, self.hi = int(lo), int(hi)

    def round_local(self, mode, rev_cap, seed) -> int:
        p = ctypes.c_int64()
        check(self.lib.knnm_round_local(self.e._h, int(mode), int(rev_cap), ctypes.c_uint64(seed),
                                        ctypes.byref(p)), "knnm_round_local")
        return int(p.value)

    def local_chunks(self) -> int:
        c = ctypes.c_int32()
        check(self.lib.knnm_local_chunks(self.e._h, ctypes.byref(c)), "knnm_local_chunks")
        return int(c.value)

    def local_join(self, chunk: int) -> None:
        check(self.lib.knnm_local_join(self.e._h, int(chunk)), "knnm_local_join")

    def local_views(self, n):
        """(cnt u32 (n,), boff u64 (n+1,), Bd f64, Bs i32) as torch views."""
        cnt, boff, bd, bs = (ctypes.c_void_p() for _ in range(4))
        check(self.lib.knnm_local_views(self.e._h, ctypes.byref(cnt), ctypes.byref(boff),
                                        ctypes.byref(bd), ctypes.byref(bs)), "knnm_local_views")
        self.e.sync()
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
        self.e.wait_torch()  # the received blocks were assembled on torch's stream
        check(self.lib.knnm_round_apply(
            self.e._h, len(base), ctypes.c_void_p(recv_cnt.data_ptr()),
            base.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(recv_bd.data_ptr()),
            ctypes.c_void_p(recv_bs.data_ptr()), ctypes.byref(acc)), "knnm_round_apply")
        return int(acc.value)

    def pack_rows(self, all_rows: bool):
        """(uint8 device view of the packed row records, count, record bytes)."""
        buf = ctypes.c_void_p()
        cnt = ctypes.c_int64()
        rb = ctypes.c_int32()
        check(self.lib.knnm_pack_rows(self.e._h, int(bool(all_rows)), ctypes.byref(buf),
                                      ctypes.byref(cnt), ctypes.byref(rb)), "knnm_pack_rows")
        self.e.signal_torch()  # torch reads the records after the pack kernel
        m, r = int(cnt.value), int(rb.value)
        return _view(buf.value, (m * r,), "|u1", self.device), m, r

    def unpack_rows(self, buf, count: int) -> None:
        if count == 0:
            return
        self.e.wait_torch()
        check(self.lib.knnm_unpack_rows(self.e._h, ctypes.c_void_p(buf.data_ptr()), int(count)),
              "knnm_unpack_rows")
        # later torch work (and the allocator's reuse of buf) is ordered
        # after the unpack kernel
        self.e.signal_torch()

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

def _as_bytes(t):
    """A flat uint8 view of a contiguous tensor, padded to 8 bytes."""
    import torch

    b = t.contiguous().reshape(-1).view(torch.uint8)
    pad = (-b.numel()) % 8
    if pad:
        b = torch.cat([b, torch.zeros(pad, dtype=torch.uint8, device=b.device)])
    return b


def _from_bytes(b, dtype, numel):
    return b[: numel * _itemsize(dtype)].view(dtype)


def _itemsize(dtype):
    import torch

    return torch.empty(0, dtype=dtype).element_size()


class LoopbackComm:
    """P virtual ranks in one process (all local)."""

    def __init__(self, world: int):
        self.world = int(world)
        self.local_ranks = list(range(self.world))

    def exchange(self, sends, extra):
        """sends[s][q] = list of tensors for rank q; returns (recv, max extra)
        with recv[q][s] = rank s's tensors for q (copies: the senders' slot
        buffers are reused by the next chunk)."""
        recv = {q: [[None if t is None else t.clone() for t in sends[s][q]]
                    for s in range(self.world)] for q in self.local_ranks}
        return recv, max(int(extra[r]) for r in self.local_ranks)

    def allgather_counts(self, vals):
        """vals[r] = list of ints; returns an int64 array (world, m)."""
        return np.array([list(vals[r]) for r in range(self.world)], dtype=np.int64)

    def allgather_bytes(self, bufs, counts, rec):
        """bufs[r] = uint8 tensor of counts[r] records; returns out[q][s]."""
        return {q: [bufs[s] for s in range(self.world)] for q in self.local_ranks}

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
    """torch.distributed communicator (one rank per process).  NCCL moves
    device tensors directly; with gloo (CPU tests) device tensors are staged
    through host memory around each collective."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_ranks = [self.rank]
        self.staged = dist.get_backend(group) != "nccl"

    def _dev(self, like):
        return like.device

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        if self.staged and inp.is_cuda:
            o = out.cpu()
            self.dist.all_to_all_single(o, inp.cpu(), output_split_sizes=out_splits,
                                        input_split_sizes=in_splits, group=self.group)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, inp, output_split_sizes=out_splits,
                                        input_split_sizes=in_splits, group=self.group)

    def _gather(self, outs, inp):
        if self.staged and inp.is_cuda:
            o = [t.cpu() for t in outs]
            self.dist.all_gather(o, inp.cpu(), group=self.group)
            for t, s in zip(outs, o):
                t.copy_(s)
        else:
            self.dist.all_gather(outs, inp, group=self.group)

    def exchange(self, sends, extra):
        import torch

        mine = sends[self.rank]
        nparts = len(mine[0])
        # dtype / presence of each part, taken from the first non-empty send
        proto = [next((p[i] for p in mine if p[i] is not None), None) for i in range(nparts)]
        dev = next(t for t in proto if t is not None).device
        packed, hdr = [], []
        for q in range(self.world):
            row = []
            for i in range(nparts):
                t = mine[q][i]
                if t is None:
                    row.append(-1)
                    continue
                b = _as_bytes(t)
                packed.append(b)
                row.append(int(t.numel()))
            row.append(int(extra[self.rank]))
            hdr.append(row)
        h = torch.tensor(hdr, dtype=torch.int64, device=dev)
        h_out = torch.empty_like(h)
        self._a2a(h_out, h)
        h_in = h_out.cpu().numpy()  # the one host read of the exchange
        dts = [None if t is None else t.dtype for t in proto]

        def nbytes(cnt, dt):
            return 0 if cnt < 0 else (cnt * _itemsize(dt) + 7) // 8 * 8

        in_splits = [sum(nbytes(hdr[q][i], dts[i]) for i in range(nparts)) for q in range(self.world)]
        out_splits = [sum(nbytes(int(h_in[s][i]), dts[i]) for i in range(nparts))
                      for s in range(self.world)]
        inp = torch.cat(packed) if packed else torch.empty(0, dtype=torch.uint8, device=dev)
        out = torch.empty(sum(out_splits), dtype=torch.uint8, device=dev)
        self._a2a(out, inp, out_splits, in_splits)
        recv, off = [], 0
        for s in range(self.world):
            parts = []
            for i in range(nparts):
                cnt = int(h_in[s][i])
                if cnt < 0:
                    parts.append(None)
                    continue
                nb = nbytes(cnt, dts[i])
                parts.append(_from_bytes(out[off: off + nb], dts[i], cnt))
                off += nb
            recv.append(parts)
        return {self.rank: recv}, int(h_in[:, nparts].max())

    def allgather_counts(self, vals):
        import torch

        dev = "cuda" if (not self.staged and torch.cuda.is_available()) else "cpu"
        t = torch.tensor(list(vals[self.rank]), dtype=torch.int64, device=dev)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return torch.stack(outs).cpu().numpy()

    def allgather_bytes(self, bufs, counts, rec):
        import torch

        mine = bufs[self.rank]
        m = int(max(counts)) * int(rec)
        pad = torch.zeros(m, dtype=torch.uint8, device=mine.device)
        pad[: mine.numel()].copy_(mine)
        outs = [torch.empty(m, dtype=torch.uint8, device=mine.device) for _ in range(self.world)]
        self._gather(outs, pad)
        return {self.rank: [outs[s][: int(counts[s]) * int(rec)] for s in range(self.world)]}

    def allgather_blocks(self, fulls, bounds):
        """Every rank's owned row block of each (n, ...) tensor, gathered in
        place (padded to the largest block)."""
        import torch

        mx = max(hi - lo for lo, hi in bounds)
        for t in fulls[self.rank]:
            lo, hi = bounds[self.rank]
            blk = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            blk[: hi - lo].copy_(t[lo:hi])
            outs = [torch.empty_like(blk) for _ in range(self.world)]
            self._gather(outs, blk)
            for r, (a, b) in enumerate(bounds):
                if r != self.rank and b > a:
                    t[a:b].copy_(outs[r][: b - a])

    def allreduce_sum(self, vals):
        import torch

        dev = "cuda" if (not self.staged and torch.cuda.is_available()) else "cpu"
        t = torch.tensor([int(vals[self.rank])], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# replication of owned rows
# ---------------------------------------------------------------------------

def _replicate_rows(shards, comm, all_rows, stats_extra=None):
    """Pack each rank's changed (or all) owned rows, all-gather them and the
    per-rank counters, unpack the other ranks' rows.  Returns the counter
    matrix (world, 1 + len(extra)): column 0 = packed row count."""
    packed = {r: shards[r].pack_rows(all_rows) for r in comm.local_ranks}
    vals = {r: [packed[r][1]] + list((stats_extra or {}).get(r, [])) for r in comm.local_ranks}
    stats = comm.allgather_counts(vals)
    counts = stats[:, 0]
    rec = packed[comm.local_ranks[0]][2]
    if int(counts.sum()):
        recv = comm.allgather_bytes({r: packed[r][0] for r in comm.local_ranks}, counts, rec)
        for q in comm.local_ranks:
            for s in range(comm.world):
                if s != q and int(counts[s]):
                    shards[q].unpack_rows(recv[q][s], int(counts[s]))
    return stats


# ---------------------------------------------------------------------------
# sharded round loop (construct.py:111-179)
# ---------------------------------------------------------------------------

def sharded_rounds(shards, comm, n, k, mode, params, rng, counter, report, rev_cap=None,
                   compact=True, traffic=None, bounds=None):
    """_descent_rounds over P ranks.  ``shards[r]`` = ShardEngine of each
    local rank r (lists replicated, shard bounds set).  ``compact``:
    exchange only the written slots (unwritten ones can never be accepted);
    ``traffic`` (dict) accumulates per rank the slot bytes sent to other
    ranks (key r) and the row-record bytes sent (key ("rows", r))."""
    import torch

    from .construct import sample_cap

    cap = sample_cap(getattr(params, "rho", 1.0), k)
    rev_cap = cap if rev_cap is None else int(rev_cap)
    bounds = shard_bounds(n, comm.world) if bounds is None else bounds
    threshold = params.min_update_fraction * n * k
    for r in comm.local_ranks:
        shards[r].set_shard(*bounds[r])
        shards[r].e.set_sample(cap if cap < k else 0)
    rounds = []
    lead = shards[comm.local_ranks[0]].e
    idx = {r: torch.tensor([b[0] for b in bounds] + [n], dtype=torch.int64, device=shards[r].device)
           for r in comm.local_ranks}
    for it in range(1, params.max_iters + 1):
        round_seed = int(rng.integers(0, 2**63 - 1))
        pairs_l = {r: shards[r].round_local(mode, rev_cap, round_seed) for r in comm.local_ranks}
        nch_l = {r: shards[r].local_chunks() for r in comm.local_ranks}
        blocks = {q: [] for q in comm.local_ranks}  # (chunk, source, parts)
        ch, nch = 0, 1
        while ch < nch:
            sends = {}
            for r in comm.local_ranks:
                shards[r].local_join(ch)
                cnt, boff, bd, bs = shards[r].local_compact(n) if compact else shards[r].local_views(n)
                cut = boff[idx[r]].cpu().numpy()  # slot offsets at the shard bounds
                parts = []
                for q, (lo, hi) in enumerate(bounds):
                    a, b = int(cut[q]), int(cut[q + 1])
                    parts.append([cnt[lo:hi], bd[a:b], None if bs is None else bs[a:b]])
                    if traffic is not None and q != r:
                        traffic[r] = traffic.get(r, 0) + (b - a) * (8 if bs is None else 12)
                sends[r] = parts
            recv, mx = comm.exchange(sends, nch_l)
            if ch == 0:
                nch = max(mx, 1)
            for q in comm.local_ranks:
                for s in range(comm.world):
                    blocks[q].append((ch, s, recv[q][s]))
            ch += 1
        acc_l = {}
        for q in comm.local_ranks:
            # (source rank, chunk) order = ascending hood order
            order = sorted(blocks[q], key=lambda x: (x[1], x[0]))
            sizes = [int(p[2][1].numel()) for p in order]
            base = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype(np.uint64)
            dev = shards[q].device
            rc = torch.cat([p[2][0].reshape(-1) for p in order]).contiguous()
            rb = torch.cat([p[2][1].reshape(-1) for p in order]).contiguous() if sum(sizes) else \
                torch.empty(1, dtype=torch.float64, device=dev)
            packed = all(p[2][2] is None for p in order)
            rs = torch.cat([p[2][2].reshape(-1) for p in order]).contiguous() \
                if (not packed and sum(sizes)) else torch.empty(1, dtype=torch.int32, device=dev)
            acc_l[q] = shards[q].round_apply(rc, base, rb, rs)
        del blocks
        stats = _replicate_rows(shards, comm, False,
                                {r: [pairs_l[r], acc_l[r]] for r in comm.local_ranks})
        if traffic is not None:
            rec = 13 * k + 8
            for r in comm.local_ranks:
                traffic[("rows", r)] = traffic.get(("rows", r), 0) + int(stats[r, 0]) * rec
        pairs = int(stats[:, 1].sum())
        accepted = int(stats[:, 2].sum())
        if pairs > 0:
            counter.add(pairs)
        lead.phi_async(it)  # reduced on the side stream, read one round later
        if rounds:
            rounds[-1][3] = lead.phi_fetch(it - 1)
        rounds.append([it, pairs, accepted, None, counter.count])
        if accepted <= threshold:
            break
    if rounds:
        rounds[-1][3] = lead.phi_fetch(rounds[-1][0])
    if report is not None:
        for r in rounds:
            report.rounds.append(RoundStats(r[0], r[1], r[2], r[3], r[4]))
        report.converged = bool(rounds) and rounds[-1][2] <= threshold


# ---------------------------------------------------------------------------
# sharded merges: sharded initialisation, sharded rounds
# ---------------------------------------------------------------------------

def _owned_slice(rows, lo, hi):
    """[a, b) with rows[a:b] the entries of the ascending ``rows`` in [lo, hi)."""
    return int(np.searchsorted(rows, lo)), int(np.searchsorted(rows, hi))


def _graph_rows(g, a, b):
    """Rows [a, b) of a graph's arrays (numpy or device tensors), duck-typed
    for Engine.load_graph."""
    return SimpleNamespace(ids=g.ids[a:b], dists=g.dists[a:b], sizes=g.sizes[a:b], k=g.k)


def _load_owned(shards, comm, rows, g, k1):
    for r in comm.local_ranks:
        a, b = _owned_slice(rows, shards[r].lo, shards[r].hi)
        if b > a:
            shards[r].e.load_graph(rows[a:b], _graph_rows(g, a, b), k1)


def _append_random_owned(shards, comm, rows, pool, count, rng, counter):
    """merge.py:166-176: the draws for every row (identical PCG64 stream on
    every rank), inserted for the owned rows only."""
    if count <= 0 or rows.size == 0 or pool.size == 0:
        return
    m, t = pool.shape[0], int(count)
    rows32 = rows.astype(np.int32)
    if t == m or 4 * t * t >= m:
        picks = _sample_pool_rows(rng, rows.size, count, pool).astype(np.int32)
        for r in comm.local_ranks:
            a, b = _owned_slice(rows, shards[r].lo, shards[r].hi)
            if b > a:
                shards[r].e.insert_rows(rows32[a:b], count, picks[a:b].ravel())
    else:
        st0 = rng.bit_generator.state
        for i, r in enumerate(comm.local_ranks):
            if i:
                rng.bit_generator.state = st0
            e = shards[r].e
            bad = e.draws_gen(rng, m, rows.size, t)
            while bad.size:
                bad = e.draws_regen(rng, m, bad)
            a, b = _owned_slice(rows, shards[r].lo, shards[r].hi)
            e.draws_insert_range(rows32, pool.astype(np.int32), a, b)
    counter.add(rows.size * t)


def _begin_sharded(dataset, union, labels, k, metric, comm, engines, bounds):
    shards = {}
    for r in comm.local_ranks:
        e = engines[r]
        e.set_dataset(dataset.vectors, int(metric))
        e.begin(union, labels, k)
        shards[r] = ShardEngine(e)
        shards[r].set_shard(*bounds[r])
    return shards


def _finish(shards, comm, union, k, k1, metric, out_device, gather, bounds):
    """Export with the rear merge (merge_rear, graph.py:259-280).  Each rank's
    rear lists cover its owned rows, so each rank's export is authoritative
    for [lo, hi).  ``gather``: all-gather those blocks and return one
    replicated graph.  Otherwise return {local rank: graph} whose rows
    outside the rank's shard are unspecified (tree levels read only their
    own rows; ``graph.shard`` = (lo, hi))."""
    import torch

    outs = {}
    for r in comm.local_ranks:
        outs[r] = list(shards[r].e.export(merge_rear=k - k1 > 0, on_device=True))
    if gather:
        comm.allgather_blocks(outs, bounds)
        outs = {comm.local_ranks[0]: outs[comm.local_ranks[0]]}
    res = {}
    for r, (ids, dists, sizes) in outs.items():
        if not out_device:
            torch.cuda.synchronize(shards[r].e.device)
            ids, dists, sizes = ids.cpu().numpy(), dists.cpu().numpy(), sizes.cpu().numpy()
        u = KnnGraph.from_arrays(union, k, metric, ids, dists, sizes)
        u.shard = None if gather else (shards[r].lo, shards[r].hi)
        res[r] = u
    return next(iter(res.values())) if gather else res


def s_merge_sharded(dataset, g, h, params: MergeParams, comm, engines, counter=None,
                    return_report=False, out_device=False, compact=True, traffic=None,
                    gather=True, bounds=None):
    """s_merge (merge.py:195-260) over comm.world ranks; ``engines`` maps each
    local rank to an Engine.  Bit-identical to s_merge.  A rank reads only the
    rows of ``g`` / ``h`` that fall in its shard of the union (the others may
    be stubs with ``member_ids``, ``k`` and ``metric`` only).  With
    ``gather=False`` the result is {local rank: graph valid on its shard}."""
    _check_merge_inputs(dataset, g, h.member_ids, params, h)
    counter = DistanceCounter() if counter is None else counter
    rng = np.random.default_rng(params.seed)
    metric = Metric(g.metric)
    k, k1 = params.k, params.k1
    union, rows_g, rows_h = _merge_members(np.asarray(g.member_ids), np.asarray(h.member_ids))
    n = union.shape[0]
    labels = np.zeros(n, dtype=np.int8)
    labels[rows_h] = 1
    bounds = shard_bounds(n, comm.world) if bounds is None else list(bounds)
    shards = _begin_sharded(dataset, union, labels, k, metric, comm, engines, bounds)
    _load_owned(shards, comm, rows_g, g, k1)
    _load_owned(shards, comm, rows_h, h, k1)
    fill = k - k1
    _append_random_owned(shards, comm, rows_g, rows_h.astype(np.int64), min(fill, rows_h.size),
                         rng, counter)
    _append_random_owned(shards, comm, rows_h, rows_g.astype(np.int64), min(fill, rows_g.size),
                         rng, counter)
    _replicate_rows(shards, comm, True)
    report = BuildReport(phi_initial=shards[comm.local_ranks[0]].e.phi())
    sharded_rounds(shards, comm, n, k, MODE_CROSS, params.descent_params(), rng, counter, report,
                   compact=compact, traffic=traffic, bounds=bounds)
    u = _finish(shards, comm, union, k, k1, metric, out_device, gather, bounds)
    return (u, report) if return_report else u


def j_merge_sharded(dataset, g, raw_ids, params: MergeParams, comm, engines, counter=None,
                    return_report=False, out_device=False, compact=True, traffic=None,
                    gather=True, bounds=None):
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
    bounds = shard_bounds(n, comm.world) if bounds is None else list(bounds)
    shards = _begin_sharded(dataset, union, labels, k, metric, comm, engines, bounds)
    _load_owned(shards, comm, rows_g, g, k1)
    _append_random_owned(shards, comm, rows_g, rows_raw.astype(np.int64),
                         min(k - k1, rows_raw.size), rng, counter)
    from .core import sample_distinct_rows

    init = sample_distinct_rows(rng, n, k, rows_raw).astype(np.int32)
    raw32 = rows_raw.astype(np.int32)
    for r in comm.local_ranks:
        a, b = _owned_slice(rows_raw, shards[r].lo, shards[r].hi)
        if b > a:
            shards[r].e.insert_rows(raw32[a:b], k, init[a:b].ravel())
    counter.add(rows_raw.size * k)
    _replicate_rows(shards, comm, True)
    report = BuildReport(phi_initial=shards[comm.local_ranks[0]].e.phi())
    sharded_rounds(shards, comm, n, k, MODE_CROSS_OR_S2, params.descent_params(), rng, counter,
                   report, compact=compact, traffic=traffic, bounds=bounds)
    u = _finish(shards, comm, union, k, k1, metric, out_device, gather, bounds)
    return (u, report) if return_report else u


# ---------------------------------------------------------------------------
# multi-way tree merge (BASELINE config 5)
# ---------------------------------------------------------------------------

def _stub(member_ids, k, metric):
    """The part of a graph a rank outside its rows needs: ids and shape."""
    return SimpleNamespace(member_ids=member_ids, k=int(k), metric=metric, n=len(member_ids),
                           ids=None, dists=None, sizes=None)


def tree_groups(world: int):
    """[(level, [ranks])] of the pairwise tree over ``world`` = 2^L ranks, in
    creation order: level l merges groups of 2^l consecutive ranks."""
    if world < 1 or world & (world - 1):
        raise ValueError("the tree merge needs a power-of-two number of ranks")
    out = []
    size = 2
    level = 1
    while size <= world:
        for j in range(world // size):
            out.append((level, list(range(j * size, (j + 1) * size))))
        size *= 2
        level += 1
    return out


def tree_merge(dataset, graphs, member_sets, params: MergeParams, world: int, group_comm,
               engines, gather_levels=None, level_hook=None):
    """Pairwise S-Merge tree of ``world`` subgraphs, one per rank (config 5).

    Level l merges, inside each group of 2^l consecutive ranks, the left
    half's graph with the right half's, sharded over the group's ranks
    (``s_merge_sharded``); groups of one level run concurrently on disjoint
    GPUs.  ``graphs[r]``: rank r's subgraph (local ranks only);
    ``member_sets[r]``: every rank's member ids, ascending and in rank order
    (subgraph r holds ids below subgraph r+1's), so rank r owns the same
    rows at every level and no list is ever re-sharded.
    ``group_comm(level, ranks)`` returns the communicator of a group (it is
    called for every group in tree order, on every process -- the contract
    of torch's new_group) or None when no local rank belongs to it.
    ``engines[r]``: the Engine of local rank r.  ``gather_levels``: gather
    each level's result (needed when several ranks live in one process);
    default: gather only when ``group_comm`` hands out LoopbackComms.
    Returns ({local rank: final graph}, [(level, ranks, DistanceCounter)]).
    """
    cur = dict(graphs)
    ids = [np.asarray(m, dtype=np.int64) for m in member_sets]
    k = params.k
    metric = Metric(next(iter(cur.values())).metric)
    log = []
    for level, members in tree_groups(world):
        comm = group_comm(level, members)
        local = [m for m in members if m in cur]
        if comm is None or not local:
            continue
        half = len(members) // 2
        sides = []
        for side in (members[:half], members[half:]):
            mine = [m for m in side if m in cur]
            sid = np.concatenate([ids[m] for m in side])
            sides.append(cur[mine[0]] if mine else _stub(sid, k, metric))
        gather = isinstance(comm, LoopbackComm) if gather_levels is None else gather_levels
        eng = {i: engines[m] for i, m in enumerate(members) if m in cur}
        # each rank keeps its own subgraph's rows at every level
        sz = np.cumsum([0] + [ids[m].size for m in members])
        bnd = [(int(sz[i]), int(sz[i + 1])) for i in range(len(members))]
        cnt = DistanceCounter()
        out = s_merge_sharded(dataset, sides[0], sides[1], params, comm, eng, counter=cnt,
                              out_device=True, gather=gather, bounds=bnd)
        for i, m in enumerate(members):
            if m in cur:
                cur[m] = out if gather else out[i]
        log.append((level, members, cnt))
        if level_hook is not None:
            level_hook(level, members, cnt)
    return cur, log
