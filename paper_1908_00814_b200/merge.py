"""Symmetric (S-Merge) and joint (J-Merge) k-NN graph merges on B200.

Drop-in mirror of the reference's merge.py (pkg/src/knnmerge/merge.py):
``s_merge`` / ``j_merge`` keep their signatures, argument meaning, input
validation (ValueError messages included), PCG64 draw sequence, return
types and output layout.  The data path -- union gather, split/localise,
random cross appends, every local-join round, export and rear merge --
runs in libknnm.so on the GPU and is bit-identical to the reference.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from .construct import (
    MODE_CROSS,
    MODE_CROSS_OR_S2,
    BuildReport,
    DescentParams,
    _capture,
    _descent_rounds,
    _graph_from,
    _emit_captured,
    _insert_directed,
    _insert_rows,
)
from .core import DistanceCounter, Metric, sample_distinct, sample_distinct_rows
from .engine import get_engine
from .graph import KnnGraph, phi as graph_phi

logger = logging.getLogger(__name__)


@dataclass
class MergeParams:
    """Merge knobs (merge.py:40-71): k, kept fraction r (k1 = round(r*k)),
    round limit and stop fraction, seed."""

    k: int
    r: float = 0.5
    max_iters: int = 50
    min_update_fraction: float = 0.001
    seed: int = 0
    rho: float = 1.0  # sample rate (DescentParams.rho; 1.0 = the reference)

    def __post_init__(self) -> None:
        if self.k < 2:
            raise ValueError("k must be >= 2")
        if not 0.0 <= self.r <= 1.0:
            raise ValueError("r must be in [0, 1]")
        if not 0.0 < self.rho <= 1.0:
            raise ValueError("rho must be in (0, 1]")

    @property
    def k1(self) -> int:
        return int(round(self.r * self.k))

    def descent_params(self) -> DescentParams:
        return DescentParams(k=self.k, max_iters=self.max_iters,
                             min_update_fraction=self.min_update_fraction, rho=self.rho)


def _lookup_local(union_gids: np.ndarray, gids: np.ndarray) -> np.ndarray:
    return np.searchsorted(union_gids, gids).astype(np.int32)


def _ascending(a: np.ndarray) -> bool:
    return a.size < 2 or bool(np.all(a[1:] > a[:-1]))


def _overlaps(a: np.ndarray, b: np.ndarray) -> bool:
    """np.intersect1d(a, b).size > 0 for ascending unique arrays, in
    O(|b| log |a|) instead of a full sort."""
    if a.size == 0 or b.size == 0:
        return False
    if not (_ascending(a) and _ascending(b)):
        return bool(np.intersect1d(a, b).size)
    idx = np.minimum(np.searchsorted(a, b), a.size - 1)
    return bool(np.any(a[idx] == b))


def _union(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """np.union1d for disjoint ascending arrays: a linear two-run merge
    (timsort detects the runs), same result as the reference's union1d."""
    if _ascending(a) and _ascending(b):
        return np.sort(np.concatenate((a, b)), kind="stable")
    return np.union1d(a, b)


def _merge_members(a: np.ndarray, b: np.ndarray, with_overlap: bool = False,
                   labels_out: list | None = None):
    """(union, rows of a, rows of b) for disjoint ascending id arrays in one
    linear pass: np.union1d + np.searchsorted of merge.py:217-221.  With
    with_overlap, also whether a and b share an id (merge.py:181).  When the
    native path runs and ``labels_out`` is a list, the int8 merge labels
    (1 = from b, merge.py:222-223) are appended to it."""
    na, nb = a.size, b.size
    if a.dtype == np.int64 and b.dtype == np.int64:
        # native merge (libknnm.so, host threads, no GPU); it rejects inputs
        # that are not strictly ascending, which take the numpy path below
        import ctypes

        from . import _lib

        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        uni = np.empty(na + nb, dtype=np.int64)
        ra = np.empty(na, dtype=np.int32)
        rb = np.empty(nb, dtype=np.int32)
        lab = np.empty(na + nb, dtype=np.int8) if labels_out is not None else None
        nu, sh = ctypes.c_int64(), ctypes.c_int32()
        rc = _lib.load().knnm_merge_members(_lib.ptr(a), na, _lib.ptr(b), nb, _lib.ptr(uni),
                                            _lib.ptr(ra), _lib.ptr(rb), ctypes.byref(nu),
                                            ctypes.byref(sh), None if lab is None else _lib.ptr(lab))
        if rc == 0:
            if lab is not None and not sh.value:
                labels_out.append(lab)
            if with_overlap:
                return uni[: nu.value], ra, rb, bool(sh.value)
            if not sh.value:
                return uni[: nu.value], ra, rb
    if not (_ascending(a) and _ascending(b)):
        u = np.union1d(a, b)
        out = (u, _lookup_local(u, a), _lookup_local(u, b))
        return out + (bool(np.intersect1d(a, b).size),) if with_overlap else out
    top = max(int(a[-1]) if na else -1, int(b[-1]) if nb else -1) + 1
    if na and nb and int(min(a[0], b[0])) >= 0 and top <= 4 * (na + nb):
        # dense id range: O(range) marker pass instead of a sort
        mark = np.zeros(top, dtype=np.int8)
        mark[a] = 1
        mark[b] += 2
        nz = mark != 0
        pos = np.cumsum(nz, dtype=np.int32) - 1
        out = (np.flatnonzero(nz).astype(np.result_type(a, b), copy=False), pos[a], pos[b])
        shared = bool(np.any(mark[b] == 3))
        if with_overlap:
            return out + (shared,)
        if not shared:  # (shared ids keep the sort path's behaviour below)
            return out
    cat = np.concatenate((a, b))
    order = np.argsort(cat, kind="stable")
    srt = cat[order]
    inv = np.empty(order.size, dtype=np.int32)
    inv[order] = np.arange(order.size, dtype=np.int32)
    out = (srt, inv[: a.size], inv[a.size:])
    if with_overlap:
        return out + (bool(srt.size > 1 and np.any(srt[1:] == srt[:-1])),)
    return out


def _sample_pool_rows(rng, nrows: int, t: int, pool: np.ndarray) -> np.ndarray:
    """(nrows, t) distinct draws per row from ``pool`` (merge.py:146-163;
    identical PCG64 call sequence)."""
    m = pool.shape[0]
    if t > m:
        raise ValueError("cannot draw more samples than the pool holds")
    if t == m or 4 * t * t >= m:
        out = np.empty((nrows, t), dtype=np.int64)
        for u in range(nrows):
            out[u] = rng.choice(m, size=t, replace=False)
        return pool[out]
    cand = rng.integers(0, m, size=(nrows, t))
    while True:
        srt = np.sort(cand, axis=1)
        bad = (np.diff(srt, axis=1) == 0).any(axis=1)
        if not bad.any():
            return pool[cand]
        rows = np.nonzero(bad)[0]
        cand[rows] = rng.integers(0, m, size=(rows.size, t))


def _append_random(engine, rows, pool, count, rng, counter, on_pair, gids) -> None:
    """merge.py:166-176: append ``count`` random pool members to each row,
    flagged new, with exact distances (device).

    The PCG64 draws stay on the host and are made in exactly the reference's
    order (merge.py:156-163); the duplicate-row test, the pool mapping and
    the inserts run on the device.  Only rows redrawn in the previous pass
    can become (or stay) bad, so re-checking just those rows finds the same
    set np.nonzero(bad) does in the reference loop."""
    if count <= 0 or rows.size == 0 or pool.size == 0:
        return
    m = pool.shape[0]
    t = int(count)
    if t > m:
        raise ValueError("cannot draw more samples than the pool holds")
    if t == m or 4 * t * t >= m:
        picks = _sample_pool_rows(rng, rows.size, count, pool)
        _insert_rows(engine, rows.astype(np.int32), count, picks.ravel().astype(np.int32),
                     counter, on_pair, gids)
        return
    # rng.integers(0, m, size=(rows.size, t)) and the redraw loop, generated
    # on the device with numpy's exact PCG64 stream (the host generator is
    # advanced to the identical state)
    bad = engine.draws_gen(rng, m, rows.size, t)
    while bad.size:
        bad = engine.draws_regen(rng, m, bad)
    engine.draws_insert(np.asarray(rows, dtype=np.int32), np.asarray(pool, dtype=np.int32))
    counter.add(rows.size * t)
    _emit_captured(engine, on_pair, gids)


def _check_merge_inputs(dataset, g: KnnGraph, other_ids: np.ndarray, params: MergeParams,
                        other_graph: KnnGraph | None, overlap: bool | None = None,
                        ascending: bool = False) -> None:
    """merge.py:179-192, same checks and messages (``ascending``: other_ids is
    known to be strictly ascending, so its extremes are its ends)."""
    if overlap is None:
        overlap = _overlaps(np.asarray(g.member_ids), np.asarray(other_ids))
    if overlap:
        raise ValueError("subsets must be disjoint")
    if g.k != params.k:
        raise ValueError(f"graph capacity {g.k} does not match params.k={params.k}")
    if other_graph is not None:
        if other_graph.metric != g.metric:
            raise ValueError("graphs must share a metric")
        if other_graph.k != params.k:
            raise ValueError("graphs must share capacity k")
    Metric(g.metric).check_kind(dataset.kind)
    if other_ids.size:
        lo, hi = (other_ids[0], other_ids[-1]) if ascending else (other_ids.min(), other_ids.max())
        if lo < 0 or hi >= dataset.n:
            raise ValueError("ids outside the dataset")


def s_merge(dataset, g: KnnGraph, h: KnnGraph, params: MergeParams,
            counter: DistanceCounter | None = None, on_pair=None, return_report: bool = False,
            device: int | None = None, out_device: bool = False):
    """Symmetric merge of two built k-NN graphs over disjoint subsets
    (merge.py:195-260; Alg. 1 of the paper)."""
    lab_out: list = []
    union_gids, rows_g, rows_h, overlap = _merge_members(
        np.asarray(g.member_ids), np.asarray(h.member_ids), with_overlap=True, labels_out=lab_out)
    _check_merge_inputs(dataset, g, h.member_ids, params, h, overlap=overlap,
                        ascending=bool(lab_out))
    if counter is None:
        counter = DistanceCounter()
    rng = np.random.default_rng(params.seed)
    metric = Metric(g.metric)
    k = params.k
    k1 = params.k1
    n = union_gids.shape[0]
    if lab_out:
        labels = lab_out[0]
    else:
        labels = np.zeros(n, dtype=np.int8)
        labels[rows_h] = 1

    eng = get_engine(device)
    eng.set_dataset(dataset.vectors, int(metric))
    eng.begin(union_gids, labels, k)
    _capture(eng, on_pair)
    try:
        eng.load_graph(rows_g, g, k1)
        eng.load_graph(rows_h, h, k1)
        fill = k - k1
        _append_random(eng, rows_g, rows_h, min(fill, rows_h.size), rng,
                       counter, on_pair, union_gids)
        _append_random(eng, rows_h, rows_g, min(fill, rows_g.size), rng,
                       counter, on_pair, union_gids)
        report = BuildReport(phi_initial=eng.phi())
        _descent_rounds(eng, n, MODE_CROSS, k, params.descent_params(), rng, counter, on_pair,
                        union_gids, report)
        ids, dists, sizes = eng.export(merge_rear=k - k1 > 0, on_device=out_device)
    finally:
        eng.set_capture(False)
    u = _graph_from(union_gids, k, metric, ids, dists, sizes)
    if return_report:
        return u, report
    return u


def j_merge(dataset, g: KnnGraph, raw_ids, params: MergeParams,
            counter: DistanceCounter | None = None, on_pair=None, return_report: bool = False,
            device: int | None = None, out_device: bool = False):
    """Joint merge of a raw id set into a built k-NN graph
    (merge.py:263-338; Alg. 2 of the paper)."""
    raw = np.asarray(raw_ids, dtype=np.int64)
    if raw.ndim != 1 or not _ascending(raw):  # np.unique of a strictly ascending array is the array
        raw = np.unique(raw)
    # one linear native pass gives the union, both row maps, the labels and
    # whether the sets overlap (np.unique + searchsorted cost 50 ms of host
    # time per 500k + 500k merge)
    lab_out: list = []
    merged = None
    if raw.size:
        merged = _merge_members(np.asarray(g.member_ids), raw, with_overlap=True, labels_out=lab_out)
    _check_merge_inputs(dataset, g, raw, params, None, overlap=None if merged is None else merged[3],
                        ascending=True)
    if counter is None:
        counter = DistanceCounter()
    metric = Metric(g.metric)
    k = params.k
    k1 = params.k1
    eng = get_engine(device)
    if raw.size == 0:
        # trivial split / merge-sort round trip (merge.py:283-291)
        eng.set_dataset(dataset.vectors, int(metric))
        eng.begin(g.member_ids, np.zeros(g.n, dtype=np.int8), k)
        eng.load_graph(np.arange(g.n, dtype=np.int32), g, k1)
        ids, dists, sizes = eng.export(merge_rear=k - k1 > 0)
        out = _graph_from(g.member_ids.copy(), k, metric, ids, dists, sizes)
        if return_report:
            return out, BuildReport(phi_initial=graph_phi(out))
        return out
    rng = np.random.default_rng(params.seed)
    union_gids, rows_g, rows_raw = merged[:3]
    n = union_gids.shape[0]
    if k >= n:
        raise ValueError(f"k={k} must be below the union size {n}")
    if lab_out:
        labels = lab_out[0]
    else:
        labels = np.zeros(n, dtype=np.int8)
        labels[rows_raw] = 1

    eng.set_dataset(dataset.vectors, int(metric))
    eng.begin(union_gids, labels, k)
    _capture(eng, on_pair)
    try:
        eng.load_graph(rows_g, g, k1)
        _append_random(eng, rows_g, rows_raw, min(k - k1, rows_raw.size), rng,
                       counter, on_pair, union_gids)
        # raw lists start from k random draws over the whole union (merge.py:318-325)
        init = sample_distinct_rows(rng, n, k, rows_raw)  # natively, same stream
        _insert_rows(eng, rows_raw.astype(np.int32), k, init.ravel().astype(np.int32), counter,
                     on_pair, union_gids)
        report = BuildReport(phi_initial=eng.phi())
        _descent_rounds(eng, n, MODE_CROSS_OR_S2, k, params.descent_params(), rng, counter,
                        on_pair, union_gids, report)
        ids, dists, sizes = eng.export(merge_rear=k - k1 > 0, on_device=out_device)
    finally:
        eng.set_capture(False)
    u = _graph_from(union_gids, k, metric, ids, dists, sizes)
    if return_report:
        return u, report
    return u


def merge_rear(u: KnnGraph, tail: KnnGraph, device: int | None = None) -> KnnGraph:
    """Per-vertex sorted merge of u's lists with rear lists, truncated to k
    (graph.py:259-280, _kernels.py:529-563), on the device."""
    if not np.all(np.isin(tail.member_ids, u.member_ids)):
        raise ValueError("tail vertices must be members of the merged graph")
    if tail.k > u.k:
        # rows are sorted by (dist, id): a wider rear list only ever
        # contributes its first u.k entries to a k-entry merged row
        # (merge_rear_rows stops at k, _kernels.py:529-563)
        narrow = KnnGraph(tail.member_ids, u.k, tail.metric)
        narrow.ids = np.ascontiguousarray(np.asarray(tail.ids)[:, : u.k])
        narrow.dists = np.ascontiguousarray(np.asarray(tail.dists)[:, : u.k])
        narrow.sizes = np.minimum(np.asarray(tail.sizes), u.k).astype(np.int32)
        tail = narrow
    eng = get_engine(device)
    # the engine needs a dataset that covers the member ids; rear merging
    # never reads vectors, so a one-column placeholder is enough
    need = int(u.member_ids[-1]) + 1 if u.n else 1
    if eng._vectors is None or eng._vectors.shape[0] < need:
        eng.set_dataset(np.zeros((need, 1), dtype=np.float32), int(u.metric))
    eng.begin(u.member_ids, np.zeros(u.n, dtype=np.int8), u.k)
    eng.load_graph(np.arange(u.n, dtype=np.int32), u, u.k)
    if tail.k > 0:
        eng.load_graph(_lookup_local(u.member_ids, tail.member_ids), tail, 0)
    ids, dists, sizes = eng.export(merge_rear=tail.k > 0)
    return _graph_from(u.member_ids.copy(), u.k, u.metric, ids, dists, sizes)
