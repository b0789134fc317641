"""Round engine and NN-Descent build on the B200 engine.

Host mirror of the reference's construct.py (pkg/src/knnmerge/construct.py).
The per-round work of ``_descent_rounds`` (construct.py:111-179) runs in one
``knnm_round`` call on the device; only the PCG64 round-seed draw, the
distance counter, the report and the convergence test stay on the host,
exactly where the reference keeps them.
"""

from __future__ import annotations

import logging
import math
from dataclasses import dataclass, field

import numpy as np

from .core import Dataset, DistanceCounter, Metric, sample_distinct
from .engine import get_engine
from .graph import KnnGraph

logger = logging.getLogger(__name__)

# Debug hook: when set to a callable, it is called as ROUND_HOOK(engine)
# after every round (tests use it for per-iteration state parity).
ROUND_HOOK = None

MODE_ALL = 0          # _kernels.py:29
MODE_CROSS = 1        # _kernels.py:30
MODE_CROSS_OR_S2 = 2  # _kernels.py:31


@dataclass
class DescentParams:
    """Knobs for NN-Descent style iteration (construct.py:31-50)."""

    k: int
    max_iters: int = 50
    min_update_fraction: float = 0.001
    # sample rate (classic NN-Descent; not in the reference, whose semantics
    # are rho = 1): per round at most ceil(rho*k) new forward entries per row
    # take part and reverse lists are capped at ceil(rho*k)
    rho: float = 1.0

    def __post_init__(self) -> None:
        if self.k < 2:
            raise ValueError("k must be >= 2")
        if not 0.0 <= self.min_update_fraction < 1.0:
            raise ValueError("min_update_fraction must be in [0, 1)")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if not 0.0 < self.rho <= 1.0:
            raise ValueError("rho must be in (0, 1]")


def sample_cap(rho: float, k: int) -> int:
    """New-entry and reverse cap per round: ceil(rho * k); k at rho = 1."""
    return k if rho >= 1.0 else max(1, int(math.ceil(rho * k)))


@dataclass
class RoundStats:
    iteration: int
    pairs: int
    updates: int
    phi: float
    distance_count: int


@dataclass
class BuildReport:
    """Per-round trace of a build or merge run (construct.py:62-76)."""

    phi_initial: float = 0.0
    rounds: list = field(default_factory=list)
    converged: bool = False

    @property
    def iterations(self) -> int:
        return len(self.rounds)

    @property
    def final_phi(self) -> float:
        return self.rounds[-1].phi if self.rounds else self.phi_initial


def _emit_captured(engine, on_pair, gids) -> None:
    """Replay the captured evaluations through the on_pair hook in reference
    order (construct.py:102-108)."""
    if on_pair is None:
        return
    pa, pb, pd = engine.fetch_captured()
    ga = gids[pa]
    gb = gids[pb]
    for a, b, d in zip(ga.tolist(), gb.tolist(), pd.tolist()):
        on_pair(int(a), int(b), float(d))


def _insert_directed(engine, rows, nids, counter, on_pair, gids) -> int:
    """_eval_pairs + apply_updates_directed (construct.py:86-108,
    _kernels.py:208-214) in one device call."""
    m = int(np.asarray(rows).shape[0])
    if m == 0:
        return 0
    acc = engine.insert_directed(rows, nids)
    counter.add(m)
    _emit_captured(engine, on_pair, gids)
    return acc


def _insert_rows(engine, rows, count, nids, counter, on_pair, gids) -> int:
    """Directed inserts with targets np.repeat(rows, count) (merge.py:173)."""
    m = int(np.asarray(nids).shape[0])
    if m == 0:
        return 0
    acc = engine.insert_rows(rows, count, nids)
    counter.add(m)
    _emit_captured(engine, on_pair, gids)
    return acc


def _descent_rounds(engine, n: int, mode: int, k: int, params, rng, counter, on_pair, gids,
                    report: BuildReport | None, rev_cap: int | None = None) -> None:
    """construct.py:111-179 on the device engine (state already loaded)."""
    threshold = params.min_update_fraction * n * k
    cap = sample_cap(getattr(params, "rho", 1.0), k)
    rev_cap = cap if rev_cap is None else int(rev_cap)
    engine.set_sample(cap if cap < k else 0)
    # phi of round `it` is reduced on a side stream while round it+1's
    # reverse / assembly / join run, and read once that round has synced
    # (the value is the same; only its report entry is completed later)
    pending = None  # (RoundStats fields of the previous round, slot)

    def flush():
        nonlocal pending
        if pending is None:
            return
        (it_, pairs_, acc_, count_), slot = pending
        cur_phi = engine.phi_fetch(slot)
        logger.info("iter=%d pairs=%d updates=%d phi=%.6f dists=%d", it_, pairs_, acc_, cur_phi, count_)
        if report is not None:
            report.rounds.append(RoundStats(it_, pairs_, acc_, cur_phi, count_))
        pending = None

    for it in range(1, params.max_iters + 1):
        round_seed = int(rng.integers(0, 2**63 - 1))
        pairs, accepted = engine.round(mode, rev_cap, round_seed)
        flush()
        if pairs > 0:
            counter.add(pairs)
        _emit_captured(engine, on_pair, gids)
        if ROUND_HOOK is not None:
            ROUND_HOOK(engine)
        engine.phi_async(it)
        pending = ((it, pairs, accepted, counter.count), it)
        if accepted <= threshold:
            flush()
            if report is not None:
                report.converged = True
            return
    flush()
    if report is not None:
        report.converged = False


def _resolve_members(dataset: Dataset, member_ids) -> np.ndarray:
    if member_ids is None:
        return np.arange(dataset.n, dtype=np.int64)
    gids = np.unique(np.asarray(member_ids, dtype=np.int64))
    if gids.size and (gids[0] < 0 or gids[-1] >= dataset.n):
        raise ValueError("member ids outside the dataset")
    return gids


def _random_lists(rng, n: int, k: int) -> np.ndarray:
    """n rows of k distinct local ids, self excluded (construct.py:192-209;
    the same PCG64 calls, so the same draws as the reference)."""
    if 4 * k * k >= n:
        from .core import sample_distinct_rows

        return sample_distinct_rows(rng, n, k, np.arange(n, dtype=np.int32))
    cand = rng.integers(0, n - 1, size=(n, k))
    cand += cand >= np.arange(n)[:, None]
    while True:
        srt = np.sort(cand, axis=1)
        bad = (np.diff(srt, axis=1) == 0).any(axis=1)
        if not bad.any():
            return cand
        rows = np.nonzero(bad)[0]
        redraw = rng.integers(0, n - 1, size=(rows.size, k))
        redraw += redraw >= rows[:, None]
        cand[rows] = redraw


def _graph_from(gids, k, metric, ids, dists, sizes) -> KnnGraph:
    """Wrap exported arrays without allocating placeholder lists; flags are
    all False like the reference's _export_graph (construct.py:212-223)."""
    return KnnGraph.from_arrays(gids, k, metric, ids, dists, sizes)


def _capture(engine, on_pair) -> None:
    engine.set_capture(on_pair is not None)


def nn_descent(dataset: Dataset, metric: Metric, params: DescentParams, seed: int,
               member_ids=None, counter: DistanceCounter | None = None, on_pair=None,
               return_report: bool = False, device: int | None = None,
               out_device: bool = False):
    """NN-Descent from a random initial graph (construct.py:226-270)."""
    metric = Metric(metric)
    metric.check_kind(dataset.kind)
    gids = _resolve_members(dataset, member_ids)
    n = gids.shape[0]
    k = params.k
    if n < 2:
        raise ValueError("need at least 2 members")
    if k >= n:
        raise ValueError(f"k={k} must be below the member count {n}")
    if counter is None:
        counter = DistanceCounter()
    rng = np.random.default_rng(seed)
    eng = get_engine(device)
    eng.set_dataset(dataset.vectors, int(metric))
    eng.begin(gids, np.zeros(n, dtype=np.int8), k)
    _capture(eng, on_pair)
    try:
        cand = _random_lists(rng, n, k)
        _insert_rows(eng, np.arange(n, dtype=np.int32), k, cand.ravel().astype(np.int32),
                     counter, on_pair, gids)
        report = BuildReport(phi_initial=eng.phi())
        _descent_rounds(eng, n, MODE_ALL, k, params, rng, counter, on_pair, gids, report)
        ids, dists, sizes = eng.export(merge_rear=False, on_device=out_device)
    finally:
        eng.set_capture(False)
    graph = _graph_from(gids, k, metric, ids, dists, sizes)
    if return_report:
        return graph, report
    return graph


def brute_force_graph(dataset: Dataset, metric: Metric, k: int, member_ids=None,
                      counter: DistanceCounter | None = None, on_pair=None,
                      device: int | None = None) -> KnnGraph:
    """Exact k-NN graph (construct.py:273-320) on the GPU.

    The reference inserts candidates in ascending id order, which makes its
    lists exactly the top-k by (fp64 distance, id); the device computes the
    same exact distances and selects by (distance, id).  With ``on_pair``
    every pair (i, j), i < j, is also handed to the hook as
    ``(gid_i, gid_j, d)`` in the reference's order (j ascending, then i;
    construct.py:296-312), the distances evaluated exactly on the device."""
    metric = Metric(metric)
    metric.check_kind(dataset.kind)
    gids = _resolve_members(dataset, member_ids)
    n = gids.shape[0]
    if k >= n:
        raise ValueError(f"k={k} must be below the member count {n}")
    if counter is None:
        counter = DistanceCounter()
    eng = get_engine(device)
    eng.set_dataset(dataset.vectors, int(metric))
    eng.begin(gids, np.zeros(n, dtype=np.int8), k)
    loc, dists = eng.bf_topk(k, rows=np.arange(n, dtype=np.int64), exclude_self=True)
    if on_pair is not None:
        _stream_all_pairs(eng, gids, on_pair)
    counter.add(n * (n - 1) // 2)
    ids = np.where(loc >= 0, gids.astype(np.int32)[np.maximum(loc, 0)], -1).astype(np.int32)
    sizes = np.full(n, min(k, n - 1), dtype=np.int32)
    return _graph_from(gids, k, metric, ids, dists, sizes)


def _stream_all_pairs(eng, gids: np.ndarray, on_pair, chunk_pairs: int = 1 << 22) -> None:
    """(gid_i, gid_j, d) for every i < j, j-major, in blocks of rows j."""
    n = gids.shape[0]
    j0 = 1
    while j0 < n:
        j1 = j0 + 1
        while j1 < n and (j1 * (j1 - 1) - j0 * (j0 - 1)) // 2 + j1 <= chunk_pairs:
            j1 += 1
        js = np.arange(j0, j1, dtype=np.int64)
        pb = np.repeat(js, js).astype(np.int32)
        starts = np.repeat(np.cumsum(js) - js, js)
        pa = (np.arange(pb.shape[0], dtype=np.int64) - starts).astype(np.int32)
        d = eng.pair_dists(pa, pb)
        ga, gb = gids[pa], gids[pb]
        for t in range(pa.shape[0]):
            on_pair(int(ga[t]), int(gb[t]), float(d[t]))
        j0 = j1


def brute_force_queries(dataset: Dataset, metric: Metric, queries: Dataset, k: int,
                        counter: DistanceCounter | None = None, device: int | None = None):
    """Exact top-k (ids int64, dists) of every query against the dataset
    (construct.py:323-348), on the GPU."""
    metric = Metric(metric)
    metric.check_kind(dataset.kind)
    metric.check_kind(queries.kind)
    if k > dataset.n:
        raise ValueError("k exceeds dataset size")
    if counter is None:
        counter = DistanceCounter()
    eng = get_engine(device)
    eng.set_dataset(dataset.vectors, int(metric))
    ids, dists = eng.bf_topk(k, queries=queries.vectors)
    counter.add(queries.n * dataset.n)
    return ids.astype(np.int64), dists
